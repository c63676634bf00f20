# same-box A/B of builds on the scoring kernel: LIBS="a.so b.so ..."; prints step time, score p50, frac
mkdir -p gpurun_out
j() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); b=d.get('breakdown_ms',{}); print('   ', sys.argv[1], round(d['ms_per_step']*1e3,1), 'us step; score p50', round(b.get('score_kernel_p50',0)*1e3,2), 'us; frac', round(d.get('roofline',{}).get('frac',0),3))" $1; }
for i in 1 2; do
for L in $LIBS; do
  echo "== $L"
  EQX_LIB=$L timeout 300 python bench.py --config cfg2 --steps 100 --warmup 10 --no-cpu-baseline --profile 2>&1 | j cfg2
  EQX_LIB=$L timeout 300 python bench.py --config cfg3 --steps 50 --warmup 10 --no-cpu-baseline --profile 2>&1 | j cfg3
done; done
