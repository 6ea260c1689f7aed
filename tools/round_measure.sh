#!/bin/bash
# One GPU-box pass of the round's measurements (run via gpurun from the repo
# root).  Outputs under gpurun_out/measure/: bench lines per config, the ncu
# launch list of the default bench command, --set full summaries of the
# dominant passes, ingest timing.  Numbers printed under ncu are never bench values.
set -u
O=gpurun_out/measure
mkdir -p $O
make -C oracle > /dev/null 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
[ -n "${SKIP_TESTS:-}" ] || { timeout 1500 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo "rc=$?" >> $O/gpu_tests.log; }
timeout 600 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
# steps per config: every timed region >= ~0.2 s, so nvidia-smi samples it
for cs in "c1 5" "c3 5" "c4 5" "c5 200" "c5ta 100"; do
  set -- $cs
  timeout 600 python bench.py --config $1 --steps $2 --warmup 3 > $O/bench_$1.json 2> $O/bench_$1.err
done
# the reference arm (the real reference package from baseline/_ref) per config
for c in c2 c1 c3 c4 c5 c5ta; do
  timeout 600 python bench.py --impl reference --config $c --steps 2 --warmup 1 > $O/bench_${c}_reference.json 2> $O/bench_${c}_reference.err
done
# launch list of the default bench command (graph-free launches: ncu cannot
# profile kernel nodes inside conditional graphs)
TS_NO_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/c2_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/c2_launches.log 2>&1
python tools/ncu_summary.py launches $O/c2_launches.csv > $O/c2_launch_shares.json 2>&1
# full captures of the dominant passes (direct pass launches via ts_time_pass)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rows_tile|k_tile_combine|k_cols_tile" -s 3 -c 3 \
  -o /tmp/c2_passes python tools/prof_pass.py c2 3 > $O/ncu_c2.log 2>&1
python tools/ncu_summary.py full /tmp/c2_passes.ncu-rep > $O/c2_full_dense_passes.json 2>&1
python tools/ncu_summary.py traffic /tmp/c2_passes.ncu-rep > $O/c2_traffic.json 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"k_rows" -s 2 -c 2 \
  -o /tmp/c4_passes python tools/prof_pass.py c4 2 > $O/ncu_c4.log 2>&1
python tools/ncu_summary.py full /tmp/c4_passes.ncu-rep > $O/c4_full_sparse_passes.json 2>&1
python tools/ncu_summary.py traffic /tmp/c4_passes.ncu-rep > $O/c4_traffic.json 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"k_rows|k_slab" -s 3 -c 3 \
  -o /tmp/c5_passes python tools/prof_pass.py c5 2 > $O/ncu_c5.log 2>&1
python tools/ncu_summary.py full /tmp/c5_passes.ncu-rep > $O/c5_full_sparse_passes.json 2>&1
python tools/ncu_summary.py traffic /tmp/c5_passes.ncu-rep > $O/c5_traffic.json 2>&1
# (the .ncu-rep files stay on the box: gpurun copies back <= 64 MiB)
timeout 600 python tools/ingest_bench.py > $O/ingest.json 2> $O/ingest.err
for c in c2 c4 c5; do python tools/prof_pass.py $c 30; done > $O/pass_times.log 2>&1
timeout 900 python tools/to_tolerance.py c3:100000 c1:10000 c4:400000 > $O/to_tolerance.json 2> $O/to_tolerance.err
timeout 600 python tools/class_breakdown.py c1:2000 c3:2000 c4:600 c2:23 > $O/class_breakdown.txt 2>&1
echo done > $O/DONE
