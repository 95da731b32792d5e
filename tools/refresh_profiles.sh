#!/bin/bash
# One GPU call: every bench line, the reference arm, launch lists and the ncu
# capture of the c4 kernel-space Gram.  Outputs under gpurun_out/refresh/.
set -u
O=gpurun_out/refresh
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
for c in 2 0 1 3 4; do
  timeout 600 python bench.py --config $c > $O/bench_c$c.log 2>&1
done
timeout 600 python bench.py --impl reference > $O/bench_reference.log 2>&1
for s in 1 3 5; do
  for c in 0 1; do
    echo "c$c streams=$s $(NYS_EIG_STREAMS=$s timeout 300 python bench.py --config $c --no-cpu-baseline 2>&1 | tail -1)" >> $O/streams.log
  done
done
for c in 1 2 4; do
  ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
      --log-file $O/launches_c$c.csv python bench.py --config $c --no-cpu-baseline --steps 3 --warmup 3 > $O/ncu_launch_c$c.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:large_kspace -s 3 -c 1 \
    -o $O/c4_kspace python bench.py --config 4 --no-cpu-baseline --steps 1 --warmup 3 > $O/ncu_full_c4.log 2>&1
