#!/bin/bash
# Round-2 evidence in one GPU call (outputs under gpurun_out/r02/): the default
# bench line (c2 + the other four configs under "configs"), the reference arm,
# launch lists of c2 / c3 / c4, ncu --set full of the c3 ladder kernel and the
# c2 batched Gram.
set -u
O=gpurun_out/r02
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
for c in 2 3 4; do
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file $O/launches_c$c.csv python bench.py --config $c --no-configs --no-cpu-baseline \
      --no-parity --steps 2 --warmup 3 > $O/ncu_launch_c$c.log 2>&1
done
# full captures: reports stay in /tmp on the box; raw + details CSV exports come back
for spec in "3:newton_ladder:0" "2:batch_gram:2" "4:large_kspace:3"; do
  IFS=: read c k s <<< "$spec"
  ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c 1 \
      -o /tmp/r02_c$c python bench.py --config $c --no-configs --no-cpu-baseline --no-parity \
      --steps 1 --warmup 3 > $O/ncu_full_c$c.log 2>&1
  ncu -i /tmp/r02_c$c.ncu-rep --page raw --csv > $O/ncu_full_c$c.raw.csv 2>/dev/null
  ncu -i /tmp/r02_c$c.ncu-rep --page details --csv > $O/ncu_full_c$c.details.csv 2>/dev/null
  ls -la /tmp/r02_c$c.ncu-rep >> $O/ncu_full_c$c.log
done
echo done
