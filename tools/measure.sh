#!/bin/bash
# Round-1 measurement pass (profiles/r01_*; superseded by tools/measure_r02.sh).  Run under gpurun; writes gpurun_out/meas/
set -u
OUT=gpurun_out/meas; mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
lscpu > $OUT/lscpu.txt 2>&1
timeout 900 python bench.py > $OUT/bench_cfg2.json 2> $OUT/bench_cfg2.err; echo "bench cfg2 rc=$?"
for c in 1 3 4 5; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 --cpu-budget 6 > $OUT/bench_cfg$c.json 2> $OUT/bench_cfg$c.err; echo "bench cfg$c rc=$?"; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref_cfg2.json 2> $OUT/bench_ref.err; echo "ref rc=$?"
# launch list of the bench command (cold-cache, serialised: compare shares)
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-twoscan --no-layered > $OUT/bench_plain.json 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_cfg2.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-twoscan --no-layered > $OUT/ncu_launch.log 2>&1; echo "launches rc=$?"
for c in 2 4 5; do
  K=k_resident; [ $c -ge 4 ] && K=k_stream_pipe
  timeout 300 python tools/prof_decode.py --config $c --reps 2 > $OUT/prof_plain_cfg$c.log 2>&1 && \
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$K -s 1 -c 1 -o $OUT/prof_cfg$c \
    python tools/prof_decode.py --config $c --reps 2 > $OUT/ncu_cfg$c.log 2>&1; echo "ncu cfg$c rc=$?"
  # summarise on the box (the full reports exceed what gpurun copies back)
  python tools/ncu_summary.py raw $OUT/prof_cfg$c.ncu-rep $OUT/ncu_full_cfg$c.json > /dev/null 2>&1 && rm -f $OUT/prof_cfg$c.ncu-rep
done
# two-scan baseline launch list (cfg2): per-kernel time and DRAM bytes
timeout 300 python tools/prof_decode.py --config 2 --sched 1 --reps 1 > /dev/null 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 \
  --csv --log-file $OUT/twoscan_cfg2.csv python tools/prof_decode.py --config 2 --sched 1 --reps 1 > /dev/null 2>&1
echo "twoscan launches rc=$?"
