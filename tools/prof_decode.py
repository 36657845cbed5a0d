#!/usr/bin/env python
"""Minimal decode driver for ncu / compute-sanitizer: decodes one BASELINE config
`--reps` times on cuda:0 (no oracle, no e2e) and prints per-launch timing."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import ldpcgen as g  # noqa: E402
import paper_cs_0609090_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--frames", type=int, default=0)
    ap.add_argument("--reps", type=int, default=4)
    ap.add_argument("--sched", type=int, default=0, help="0 single-scan, 1 two-scan, 2 layered")
    ap.add_argument("--full", action="store_true", help="LDPC_MSG_FULL (the §4 per-edge message form)")
    ap.add_argument("--f32", action="store_true", help="decode the config's LLRs as fp32 (normalized 0.75)")
    args = ap.parse_args()
    cfg = g.CONFIGS[args.config]
    code = cfg.code()
    F = args.frames or cfg.frames
    llr = torch.from_numpy(cfg.llrs(code, 0, F)).cuda()
    dec = P.Decoder(code, 0)
    params = P.params_for_config(cfg, schedule=args.sched, msg_format=P.LDPC_MSG_FULL if args.full else None)
    if args.f32:
        llr = llr.float()
        params = P.make_params(cfg.max_iter, 0, P.LDPC_MINSUM_NORMALIZED, 0, 0.0, 0.75, 0, P.LDPC_LLR_F32,
                               P.LDPC_MSG_COMPACT)
    out = dec.alloc_outputs(F, params.llr_type, posteriors=True)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for i in range(args.reps):
        ev[0].record()
        dec.decode(llr, params, out)
        ev[1].record()
        torch.cuda.synchronize()
        print(f"rep {i}: {ev[0].elapsed_time(ev[1]):.3f} ms, launches {P.ldpc_last_launch_count()}", flush=True)


if __name__ == "__main__":
    main()
