#!/bin/bash
# Round-2 measurement pass on one B200 (run under gpurun); writes gpurun_out/meas/.
set -u
OUT=gpurun_out/meas; mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
lscpu > $OUT/lscpu.txt 2>&1
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref rc=$?"
# launch list of the headline bench command (cold-cache, serialised: compare shares)
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-twoscan --no-layered --no-per-config --no-e2e \
  > $OUT/bench_plain.json 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_cfg2.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-twoscan --no-layered --no-per-config --no-e2e \
  > $OUT/ncu_launch.log 2>&1; echo "launches rc=$?"
for c in 1 2 3 4 5; do
  K=k_resident_atom; S=1; FR=""; [ $c -ge 4 ] && K=k_stream_pipe && S=3
  [ $c -eq 3 ] && FR="--frames 16384"; [ $c -eq 5 ] && FR="--frames 1024"
  timeout 300 python tools/prof_decode.py --config $c $FR --reps 2 > $OUT/prof_plain_cfg$c.log 2>&1 && \
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$K -s $S -c 1 -o $OUT/prof_cfg$c \
    python tools/prof_decode.py --config $c $FR --reps 2 > $OUT/ncu_cfg$c.log 2>&1; echo "ncu cfg$c rc=$?"
  python tools/ncu_summary.py raw $OUT/prof_cfg$c.ncu-rep $OUT/ncu_full_cfg$c.json > /dev/null 2>&1
  ncu -i $OUT/prof_cfg$c.ncu-rep --page source --csv > $OUT/ncu_source_cfg$c.csv 2>/dev/null
  rm -f $OUT/prof_cfg$c.ncu-rep
done
