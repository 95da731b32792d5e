#!/bin/bash
# Round-2 (session 3) evidence in one GPU call (outputs under gpurun_out/r02b/):
# the default bench line (c2 + the other four configs under "configs"), the
# reference arm, launch lists of every config, ncu --set full exports of the
# c2 batched Gram, the c3 ladder, the c4 kernel-space Gram and the cluster
# eigensolver (raw + details CSV come back; the .ncu-rep stay on the box).
set -u
O=gpurun_out/${R02_OUT:-r02d}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
for c in 0 1 2 3 4; do
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file $O/launches_c$c.csv python bench.py --config $c --no-configs --no-cpu-baseline \
      --no-parity --steps 2 --warmup 3 > $O/ncu_launch_c$c.log 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/launches_eig256.csv python tools/eig_one.py 4 > $O/ncu_launch_eig.log 2>&1
for spec in "3:newton_ladder:0" "2:batch_gram:2" "4:large_kspace:3"; do
  IFS=: read c k s <<< "$spec"
  ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c 1 \
      -o /tmp/r02b_c$c python bench.py --config $c --no-configs --no-cpu-baseline --no-parity \
      --steps 1 --warmup 3 > $O/ncu_full_c$c.log 2>&1
  ncu -i /tmp/r02b_c$c.ncu-rep --page raw --csv > $O/ncu_full_c$c.raw.csv 2>/dev/null
  ncu -i /tmp/r02b_c$c.ncu-rep --page details --csv > $O/ncu_full_c$c.details.csv 2>/dev/null
done
ncu --set full --clock-control none --import-source on -k regex:dcc_eig -c 1 \
    -o /tmp/r02b_eig python tools/eig_one.py 4 > $O/ncu_full_eig.log 2>&1
ncu -i /tmp/r02b_eig.ncu-rep --page raw --csv > $O/ncu_full_eig.raw.csv 2>/dev/null
ncu -i /tmp/r02b_eig.ncu-rep --page details --csv > $O/ncu_full_eig.details.csv 2>/dev/null
NYS_EIG_DEBUG=1 python tools/eig_one.py 4 > $O/eig_phases.txt 2>&1
python tools/c4_rank_model.py > $O/c4_rank_model.jsonl 2> $O/c4_rank_model.err
echo done
