#!/usr/bin/env python
"""Sweep the resident CTA size for config 1 (general code, barrier-free kernel): time a CUDA
graph of 64 decodes of distinct 1024-frame batches per thread count."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import ldpcgen as g  # noqa: E402
import paper_cs_0609090_b200 as P  # noqa: E402

cfg = g.CONFIGS[1]
code = cfg.code()
F = cfg.frames
NB = 64
dec = P.Decoder(code, 0)
batches = [torch.from_numpy(cfg.llrs(code, 1_000_000 * (b + 1), F)).cuda() for b in range(NB)]
for th in [int(x) for x in (sys.argv[1:] or [0, 64, 96, 128, 160, 192, 224, 256])]:
    params = P.params_for_config(cfg)
    if th:
        P.set_tuning(params, {"resident_threads": th})
    outs = [dec.alloc_outputs(F, params.llr_type) for _ in range(NB)]
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for b in range(NB):
            dec.decode(batches[b], params, outs[b])
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=s):
        for b in range(NB):
            dec.decode(batches[b], params, outs[b])
    ts = []
    for _ in range(8):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        gr.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / NB)
    print(f"threads {th}: {min(ts):.4f} ms/decode (median {sorted(ts)[4]:.4f})", flush=True)
