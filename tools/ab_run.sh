# same-box A/B of builds: LIBS="a.so b.so ..." (default: ab/libeqx_old.so and the in-tree library);
# CFGS selects the workloads (default: cfg4 simulated global, cfg2, cfg3); NOTEST=1 skips pytest
mkdir -p gpurun_out
[ -z "$NOTEST" ] && timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
LIBS=${LIBS:-"ab/libeqx_old.so paper_2508_16646_b200/libeqx_b200.so"}
CFGS=${CFGS:-"cfg4sim cfg2 cfg3"}
j() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('   ', sys.argv[1], round(d['ms_per_step']*1e3,1), 'us', d.get('e2e',{}).get('value'))" $1; }
for i in 1 2; do
for L in $LIBS; do
  echo "== $L"
  for c in $CFGS; do
    case $c in
      cfg4sim) EQX_LIB=$L timeout 300 python bench.py --config cfg4 --simulate-world 8 --steps 50 --warmup 5 --no-cpu-baseline 2>&1 | j $c ;;
      cfg2) EQX_LIB=$L timeout 300 python bench.py --config cfg2 --steps 200 --warmup 10 --no-cpu-baseline 2>&1 | j $c ;;
      *) EQX_LIB=$L timeout 300 python bench.py --config $c --steps 100 --warmup 10 --no-cpu-baseline 2>&1 | j $c ;;
    esac
  done
done; done
