timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
for v in default 4 5 6; do
  if [ $v = default ]; then L=""; else L="SDEDGE_LIB=build_variants/libsdedge_minb$v.so"; fi
  env $L timeout 300 python bench.py --n 200000 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']), d['roofline']['frac'])"
  env $L timeout 300 python bench.py --algo dense --n 20000 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v dense', round(d['value']), d['roofline']['frac'])"
done
