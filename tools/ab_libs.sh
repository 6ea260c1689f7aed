# A/B of two builds of the library on the same box: device it/s per config,
# alternating the libraries (TS_LIB_PATH).  usage: tools/ab_libs.sh libA.so libB.so
A=$1; B=$2; O=gpurun_out/ab; mkdir -p $O
for rep in 1 2; do
  for c in ${CFGS:-c5:200 c5ta:100 c4:5 c3:5 c1:3}; do
    cfg=${c%%:*}; st=${c##*:}
    for L in A B; do
      lib=$A; [ $L = B ] && lib=$B
      TS_LIB_PATH=$PWD/$lib timeout 300 python bench.py --config $cfg --steps $st --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$cfg $L rep$rep', round(d['value'],1), {k:round(v['avg_us'],2) for k,v in d['kernel_breakdown'].items() if 'avg_us' in v})"
    done
  done
done | tee $O/ab.txt
