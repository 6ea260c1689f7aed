# one GPU pass: the device tests (optionally a subset), then bench lines
set -x
T=${TESTS:-tests}
timeout 1500 python -m pytest $T -m gpu -x -q -s ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -40 > gpurun_out/gputests.txt
for c in ${CONFIGS:-}; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
cat gpurun_out/gputests.txt
