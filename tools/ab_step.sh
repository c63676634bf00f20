# same-box A/B of builds on the step: LIBS="a.so b.so ..."; step time, drain p50, score p50 per config
mkdir -p gpurun_out
j() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); b=d.get('breakdown_ms',{}); print('   ', sys.argv[1], round(d['ms_per_step']*1e3,1), 'us step; drain p50', round(b.get('drain_p50',0)*1e3,2), '; score p50', round(b.get('score_kernel_p50',0)*1e3,2), 'us')" $1; }
for i in 1 2; do
for L in $LIBS; do
  echo "== $L"
  EQX_LIB=$L timeout 300 python bench.py --config cfg2 --steps 100 --warmup 10 --no-cpu-baseline --profile 2>&1 | j cfg2
  EQX_LIB=$L timeout 300 python bench.py --config cfg3 --steps 50 --warmup 10 --no-cpu-baseline --profile 2>&1 | j cfg3
done; done
