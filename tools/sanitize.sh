#!/bin/bash
# compute-sanitizer on small decodes of every kernel family (run under gpurun, ONE tool per
# call -- the profiling guide: several tools in one call have left GPUs unusable):
#   bash tools/sanitize.sh <memcheck|racecheck|synccheck|initcheck>
TOOL=${1:-memcheck}
mkdir -p gpurun_out
timeout 300 python tools/san_workload.py > gpurun_out/san_plain.log 2>&1 && \
timeout 1200 compute-sanitizer --tool $TOOL --print-limit 20 --error-exitcode 9 python tools/san_workload.py \
  > gpurun_out/sanitizer_$TOOL.log 2>&1
echo "sanitizer $TOOL rc=$?"
tail -5 gpurun_out/sanitizer_$TOOL.log
