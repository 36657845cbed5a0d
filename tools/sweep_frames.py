#!/usr/bin/env python
"""Decode time against batch size for the resident kernels (wave quantisation / load
balance): cfg1 timed as a CUDA graph of 32 decodes, cfg2 as single decodes (median of 7).
Usage: python tools/sweep_frames.py CFG F1 F2 ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import ldpcgen as g  # noqa: E402
import paper_cs_0609090_b200 as P  # noqa: E402


def time_cfg(c, F):
    cfg = g.CONFIGS[c]
    code = cfg.code()
    dec = P.Decoder(code, 0)
    params = P.params_for_config(cfg)
    NB = 32 if c == 1 else 1
    batches = [torch.from_numpy(cfg.llrs(code, 1_000_000 * (b + 1), F)).cuda() for b in range(NB)]
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
    for _ in range(7):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        gr.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / NB)
    return sorted(ts)[3]


if __name__ == "__main__":
    c = int(sys.argv[1])
    for F in [int(x) for x in sys.argv[2:]]:
        t = time_cfg(c, F)
        print(f"cfg{c} frames {F} pairs {F // 2}: {t:.4f} ms  ({1e3 * t / (F / 2):.3f} us per pair)", flush=True)
