#!/usr/bin/env python
"""Sweep the host-buffer decode's chunking (ldpc_tuning.host_chunks / host_streams) on a
BASELINE config: pinned host LLRs in, hard bits / posteriors / flags / iterations out.
    python tools/sweep_e2e.py CFG [CHUNKS,STREAMS ...]   (0,0 = the library's default)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import ldpcgen as g  # noqa: E402
import paper_cs_0609090_b200 as P  # noqa: E402

cfg = g.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
code = cfg.code()
F = cfg.frames
dec = P.Decoder(code, 0)
llr = cfg.llrs(code, 0, F)
lh = torch.from_numpy(llr).pin_memory()
hb = torch.empty((F, dec.wpf), dtype=torch.int32).pin_memory()
ok = torch.empty(F, dtype=torch.uint8).pin_memory()
it = torch.empty(F, dtype=torch.int32).pin_memory()
post = torch.empty((F, code.n_vars), dtype=torch.float32 if llr.dtype == np.float32 else torch.int16).pin_memory()
for chunks, streams in [(int(a), int(b)) for a, b in (x.split(",") for x in sys.argv[2:])] or [(0, 0), (1, 1), (2, 2), (2, 1), (4, 4), (8, 4), (16, 4)]:
    params = P.params_for_config(cfg)
    P.set_tuning(params, {"host_chunks": chunks, "host_streams": streams})
    for _ in range(2):
        dec.decode_host(lh, params, hb, ok, it, post)
    torch.cuda.synchronize()
    ts = []
    for _ in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dec.decode_host(lh, params, hb, ok, it, post)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[len(ts) // 2]
    import time
    torch.cuda.synchronize()
    c0 = time.perf_counter()
    for _ in range(20):
        dec.decode_host(lh, params, hb, ok, it, post)
    c1 = time.perf_counter()
    torch.cuda.synchronize()
    c2 = time.perf_counter()
    print(f"   host enqueue {(c1 - c0) / 20 * 1e3:.3f} ms/call, back-to-back {(c2 - c0) / 20 * 1e3:.3f} ms/call")
    print(f"chunks {chunks} streams {streams}: {ms:.3f} ms, {F * code.K / (ms * 1e-3) / 1e9:.2f} Gbit/s", flush=True)
