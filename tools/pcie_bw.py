#!/usr/bin/env python
"""PCIe bandwidth on the GPU box for the e2e leg's byte counts (cfg2: 123 MB of LLRs in, 131 MB
of hard bits + posteriors + flags out per step): copy engines (one copy / chunked, one or both
directions) and SM-driven zero-copy access to mapped pinned memory.  Writes
profiles/r02_pcie_bw.json.  Run on the GPU box: python tools/pcie_bw.py"""
import ctypes
import functools
import json
import os
import subprocess
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
so = os.path.join(ROOT, "build", "libpcie_copy.so")
subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler", "-fPIC",
                       "-o", so, os.path.join(ROOT, "tools", "pcie_copy.cu")])
L = ctypes.CDLL(so)
L.zc_copyw.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                       ctypes.c_void_p]
n_in, n_out = 123_000_000 // 16 * 16, 131_000_000 // 16 * 16
h_in = torch.empty(n_in, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n_out, dtype=torch.uint8).pin_memory()
d_in = torch.empty(n_in, dtype=torch.uint8, device="cuda")
d_out = torch.empty(n_out, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        fn()
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return round(sorted(ts)[len(ts) // 2], 3)


def ce_h2d(n=1):
    c = n_in // n
    for i in range(n):
        with torch.cuda.stream(s1):
            d_in[i * c:(i + 1) * c].copy_(h_in[i * c:(i + 1) * c], non_blocking=True)


def ce_d2h(n=1):
    c = n_out // n
    for i in range(n):
        with torch.cuda.stream(s2):
            h_out[i * c:(i + 1) * c].copy_(d_out[i * c:(i + 1) * c], non_blocking=True)


def sm_d2h(w=16):
    L.zc_copyw(d_out.data_ptr(), h_out.data_ptr(), n_out, 592, 256, w, s2.cuda_stream)


def sm_h2d(w=16):
    L.zc_copyw(h_in.data_ptr(), d_in.data_ptr(), n_in, 592, 256, w, s1.cuda_stream)


res = {"bytes_in": n_in, "bytes_out": n_out, "unit": "ms per transfer of both byte counts (median of 5)"}
res["ce_h2d"] = timed(ce_h2d)
res["ce_d2h"] = timed(ce_d2h)
res["ce_both_one_copy_each"] = timed(lambda: (ce_h2d(), ce_d2h()))
for n in (2, 4, 8, 16):
    res[f"ce_h2d_{n}_chunks"] = timed(functools.partial(ce_h2d, n))
    res[f"ce_both_{n}_chunks_each"] = timed(lambda: (ce_h2d(n), ce_d2h(n)))
    res[f"ce_h2d_{n}_chunks_plus_ce_d2h_one"] = timed(lambda: (ce_h2d(n), ce_d2h()))
for w in (2, 4, 16):
    res[f"sm_d2h_{w}B"] = timed(functools.partial(sm_d2h, w))
res["sm_h2d_16B"] = timed(sm_h2d)
res["ce_h2d_plus_sm_d2h"] = timed(lambda: (ce_h2d(), sm_d2h()))
res["ce_h2d_16_chunks_plus_sm_d2h"] = timed(lambda: (ce_h2d(16), sm_d2h()))
res["sm_h2d_plus_ce_d2h"] = timed(lambda: (sm_h2d(), ce_d2h()))
# the e2e pipeline's pattern (ldpc_decode_batch_host): chunk i's H2D, its decode (a
# device-side sleep of the chunk's share of the 2.28 ms cfg2 decode) and its D2H on stream
# i % 4; weights = relative chunk sizes
ss = [torch.cuda.Stream() for _ in range(4)]


def pipeline(w):
    tot, a, b = sum(w), 0, 0
    for i, x in enumerate(w):
        ci = n_in * x // tot // 16 * 16 if i < len(w) - 1 else n_in - a
        co = n_out * x // tot // 16 * 16 if i < len(w) - 1 else n_out - b
        with torch.cuda.stream(ss[i % 4]):
            d_in[a:a + ci].copy_(h_in[a:a + ci], non_blocking=True)
            torch.cuda._sleep(int(2.28e-3 * 1.9e9 * x / tot))
            h_out[b:b + co].copy_(d_out[b:b + co], non_blocking=True)
        a += ci
        b += co
    for x in ss:
        torch.cuda.current_stream().wait_stream(x)


for name, w in [("uniform_4", [1] * 4), ("uniform_8", [1] * 8), ("uniform_16", [1] * 16), ("uniform_32", [1] * 32),
                ("ramp_10", [1, 1, 2, 4, 8, 8, 4, 2, 1, 1])]:
    res[f"pipeline_{name}"] = timed(functools.partial(pipeline, w))
res["gbs_h2d"] = round(n_in / res["ce_h2d"] / 1e6, 1)
res["gbs_d2h"] = round(n_out / res["ce_d2h"] / 1e6, 1)
res["gbs_both_total"] = round((n_in + n_out) / res["ce_both_one_copy_each"] / 1e6, 1)
print(json.dumps(res))
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", "pcie_bw.json"), "w") as f:
    json.dump(res, f, indent=1)
