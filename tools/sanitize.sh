#!/bin/bash
# compute-sanitizer on small decodes (run under gpurun, one tool per call): sanitize.sh <tool>
TOOL=${1:-memcheck}
cat > /tmp/san_run.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import ldpcgen as g, paper_cs_0609090_b200 as P
for idx, F in ((1, 9), (2, 6), (3, 5)):
    cfg = g.CONFIGS[idx]; code = cfg.code()
    d = P.Decoder(code, 0); out = d.decode(torch.from_numpy(cfg.llrs(code, 0, F)).cuda(), P.params_for_config(cfg))
    torch.cuda.synchronize()
os.environ["LDPC_FORCE_STREAM"] = "1"
code = g.regular(96, 3, 6, seed=5)
for kind, pt in ((g.LLR_I16, P.LDPC_LLR_I16),):
    d = P.Decoder(code, 0)
    llr = g.llr(3, 0, 70, 96, 0.8, kind, 3, 511)
    d.decode(torch.from_numpy(llr).cuda(), P.make_params(6, 1, 0, 1, 0, 1.0, 511, pt)); torch.cuda.synchronize()
llr = g.llr(3, 0, 40, 96, 0.8, g.LLR_F32)
d.decode(torch.from_numpy(llr).cuda(), P.make_params(6, 1, 1, 0, 0, 0.75, 0, P.LDPC_LLR_F32)); torch.cuda.synchronize()
print("sanitizer workload done")
PY
python /tmp/san_run.py > gpurun_out/san_plain.log 2>&1 && \
timeout 1200 compute-sanitizer --tool $TOOL --print-limit 20 python /tmp/san_run.py > gpurun_out/sanitizer_$TOOL.log 2>&1
echo "sanitizer $TOOL rc=$?"
tail -5 gpurun_out/sanitizer_$TOOL.log
