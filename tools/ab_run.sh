
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for i in 1 2; do
for L in ab/libeqx_old.so paper_2508_16646_b200/libeqx_b200.so; do
  echo "== $L"
  EQX_LIB=$L timeout 300 python bench.py --config cfg4 --simulate-world 8 --steps 50 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d.get('e2e',{}).get('value'))"
  EQX_LIB=$L timeout 300 python bench.py --config cfg2 --steps 200 --warmup 10 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d.get('e2e',{}).get('value'))"
  EQX_LIB=$L timeout 300 python bench.py --config cfg3 --steps 100 --warmup 10 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d.get('e2e',{}).get('value'))"
done; done
