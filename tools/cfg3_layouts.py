#!/usr/bin/env python
"""Config 3 (1-bit messages, 65536 frames, 30 iterations) on the resident kernel (lanes = check
rows; a frame pair per CTA, sign bits of a row-pair packed per lane) against the streaming
kernel (lanes = frame pairs, 64 frames per warp tile, state through HBM) -- the measurement
behind DESIGN.md's choice of layout for the 1-bit format."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import ldpcgen as g  # noqa: E402
import paper_cs_0609090_b200 as P  # noqa: E402

cfg = g.CONFIGS[3]
code = cfg.code()
F = cfg.frames
llr = torch.from_numpy(cfg.llrs(code, 0, F)).cuda()
dec = P.Decoder(code, 0)
res = {"workload": f"cfg3, {F} frames, {cfg.max_iter} iterations"}
for name, tn in (("resident", None), ("streaming", {"path": P.LDPC_PATH_STREAM})):
    params = P.params_for_config(cfg)
    if tn:
        P.set_tuning(params, tn)
    out = dec.alloc_outputs(F, params.llr_type)
    for _ in range(2):
        dec.decode(llr, params, out)
    torch.cuda.synchronize()
    ts = []
    for _ in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dec.decode(llr, params, out)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = min(ts)
    res[name] = {"ms_per_decode": ms, "info_gbps": F * code.K / (ms * 1e-3) / 1e9,
                 "edge_updates_per_s": F * cfg.max_iter * code.n_edges / (ms * 1e-3),
                 "launches": P.ldpc_last_launch_count()}
print(json.dumps(res))
