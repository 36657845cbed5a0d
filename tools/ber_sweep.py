#!/usr/bin/env python
"""BER / FER sweep over Eb/N0 with the GPU decoder.

The paper prints no BER/FER curves (its experiment is speed only), so these numbers
are reported, never asserted.  Frames: all-zero codeword, BPSK over AWGN from the
seeded generator (ldpcgen); errors counted on the GPU (ldpc_count_errors, reading
D14).  Example:

    python tools/ber_sweep.py --config 2 --ebn0 1.0 1.5 2.0 2.5 3.0 --frames 8192 \
        --schedule singlescan layered
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import ldpcgen as g  # noqa: E402
import paper_cs_0609090_b200 as P  # noqa: E402

SCHED = {"singlescan": P.LDPC_SCHED_SINGLESCAN, "twoscan": P.LDPC_SCHED_TWOSCAN, "layered": P.LDPC_SCHED_LAYERED}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--ebn0", type=float, nargs="+", default=[1.0, 1.5, 2.0, 2.5, 3.0])
    ap.add_argument("--frames", type=int, default=4096)
    ap.add_argument("--seed", type=int, default=7001)
    ap.add_argument("--schedule", nargs="+", default=["singlescan"], choices=list(SCHED))
    ap.add_argument("--max-iter", type=int, default=0, help="override the config's iteration cap")
    ap.add_argument("--early-stop", type=int, default=-1, help="override early stop (0/1)")
    args = ap.parse_args()
    cfg = g.CONFIGS[args.config]
    if args.max_iter:
        cfg.max_iter = args.max_iter
    if args.early_stop >= 0:
        cfg.early_stop = args.early_stop
    code = cfg.code()
    dec = P.Decoder(code, 0)
    frac = {g.LLR_I16: 3, g.LLR_I8: 2}.get(cfg.llr_kind, 0)
    rows = []
    for eb in args.ebn0:
        s2 = g.ebn0_to_sigma2(eb, code.rate)
        llr = g.llr(args.seed, 0, args.frames, code.n_vars, s2, cfg.llr_kind, frac, cfg.clamp) if frac else \
            g.llr(args.seed, 0, args.frames, code.n_vars, s2, cfg.llr_kind)
        t = torch.from_numpy(llr).cuda()
        for sname in args.schedule:
            params = P.params_for_config(cfg, SCHED[sname])
            try:
                out = dec.decode(t, params, posteriors=False)
            except P.LdpcError as e:
                rows.append({"ebn0_db": eb, "schedule": sname, "unsupported": str(e)})
                continue
            c = dec.count_errors(out).cpu().tolist()
            F, N = args.frames, code.n_vars
            rows.append({"ebn0_db": eb, "schedule": sname, "frames": F, "ber": c[0] / (F * N), "fer": c[1] / F,
                         "undetected": c[2], "not_converged": c[3], "mean_iterations": c[4] / F})
            print(json.dumps(rows[-1]), flush=True)
    print(json.dumps({"config": cfg.idx, "code": code.name, "rate": code.rate, "max_iter": cfg.max_iter,
                      "early_stop": cfg.early_stop, "points": rows}))


if __name__ == "__main__":
    main()
