#!/usr/bin/env python
"""Small decodes over every kernel family, for compute-sanitizer (tools/sanitize.sh):
resident barrier-free (CSR, QC, 1-bit, FULL, message export), resident batched and
layered (int16, fp32), streaming (int16 + early stop, 1-bit, fp32 pipelined and register
kernels, message export) and the two-scan baseline."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import ldpcgen as g  # noqa: E402
import paper_cs_0609090_b200 as P  # noqa: E402


def run(code, llr, params, msgs=False):
    d = P.Decoder(code, 0)
    t = torch.from_numpy(llr).cuda()
    if msgs:
        d.decode_messages(t, params)
    else:
        d.decode(t, params)
    torch.cuda.synchronize()
    d.close()


for idx, F in ((1, 9), (2, 6), (3, 5)):
    cfg = g.CONFIGS[idx]
    code = cfg.code()
    llr = cfg.llrs(code, 0, F)
    run(code, llr, P.params_for_config(cfg))
    run(code, llr, P.params_for_config(cfg), msgs=True)
    run(code, llr, P.params_for_config(cfg, P.LDPC_SCHED_LAYERED))
    if idx != 3:
        run(code, llr, P.params_for_config(cfg, msg_format=P.LDPC_MSG_FULL), msgs=True)
        run(code, llr, P.set_tuning(P.params_for_config(cfg), {"path": P.LDPC_PATH_RESIDENT_BATCHED}))
code = g.regular(96, 3, 6, seed=5)
i16 = g.llr(3, 0, 70, 96, 0.8, g.LLR_I16, 3, 511)
i8 = g.llr(4, 0, 70, 96, 0.8, g.LLR_I8, 2, 127)
f32 = g.llr(5, 0, 40, 96, 0.8, g.LLR_F32)
ST = {"path": P.LDPC_PATH_STREAM}
run(code, i16, P.make_params(6, 1, 0, 1, 0, 1.0, 511, P.LDPC_LLR_I16, tuning=ST))
run(code, i16, P.make_params(6, 0, 0, 1, 0, 1.0, 511, P.LDPC_LLR_I16, tuning=ST), msgs=True)
run(code, i8, P.make_params(6, 1, 0, 1, 0, 1.0, 127, P.LDPC_LLR_I8, P.LDPC_MSG_1BIT, tuning=ST))
run(code, f32, P.make_params(6, 1, 1, 0, 0, 0.75, 0, P.LDPC_LLR_F32))
run(code, f32, P.make_params(6, 0, 1, 0, 0, 0.75, 0, P.LDPC_LLR_F32), msgs=True)
run(code, f32, P.make_params(6, 1, 1, 0, 0, 0.75, 0, P.LDPC_LLR_F32, tuning={"stream_register_kernels": 1}))
run(code, f32, P.make_params(6, 1, 1, 0, 0, 0.75, 0, P.LDPC_LLR_F32, P.LDPC_MSG_COMPACT, P.LDPC_SCHED_LAYERED))
run(code, i16, P.make_params(6, 1, 0, 1, 0, 1.0, 511, P.LDPC_LLR_I16, P.LDPC_MSG_COMPACT, P.LDPC_SCHED_TWOSCAN),
    msgs=True)
run(code, f32, P.make_params(6, 1, 1, 0, 0, 0.75, 0, P.LDPC_LLR_F32, P.LDPC_MSG_COMPACT, P.LDPC_SCHED_TWOSCAN))
print("sanitizer workload done")
