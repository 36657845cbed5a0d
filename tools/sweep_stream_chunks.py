#!/usr/bin/env python
"""Streaming kernels (cfg4 int16, cfg5 fp32): decode time against ldpc_tuning.stream_chunk_tiles
(frame tiles decoded together through all iterations; 0 = all tiles at once).  Small chunks
keep a chunk's planes in the 126 MB L2 across iterations -- if the kernels were bound by DRAM
bytes this would pay.  Writes gpurun_out/stream_chunks.json.  Run on the GPU box."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import ldpcgen as g  # noqa: E402
import paper_cs_0609090_b200 as P  # noqa: E402

res = {"unit": "ms per decode (median of 5)"}
for idx, F in ((4, g.CONFIGS[4].frames), (5, 1024)):
    cfg = g.CONFIGS[idx]
    code = cfg.code()
    dec = P.Decoder(code, 0)
    llr = torch.from_numpy(cfg.llrs(code, 0, F)).cuda()
    for ct in (0, 1, 2, 4):
        p = P.params_for_config(cfg)
        P.set_tuning(p, {"stream_chunk_tiles": ct})
        out = dec.alloc_outputs(F, p.llr_type, posteriors=True)
        dec.decode(llr, p, out)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            dec.decode(llr, p, out)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        res[f"cfg{idx}_F{F}_chunk_tiles_{ct}"] = round(sorted(ts)[2], 3)
        print(f"cfg{idx} F={F} chunk_tiles={ct}: {sorted(ts)[2]:.3f} ms", flush=True)
    dec.close()
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", "stream_chunks.json"), "w") as f:
    json.dump(res, f, indent=1)
