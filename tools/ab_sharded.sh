j() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('   ', sys.argv[1], round(d['ms_per_step']*1e3,1), 'us step', d.get('breakdown_ms'))" $1; }
for i in 1 2; do for L in ab/libeqx_old.so ab/libeqx_sh.so; do echo "== $L";
EQX_LIB=$L timeout 300 python bench.py --config cfg4 --steps 50 --warmup 5 --no-cpu-baseline --profile 2>&1 | j cfg4
EQX_LIB=$L timeout 300 python bench.py --config cfg4 --simulate-world 8 --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | j sim8
done; done
