timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python tools/paper_context.py --n 2000 > gpurun_out/r01_paper_context.json 2> gpurun_out/paper_context.err; echo rc=$?
python -c "
import json; d=json.load(open('gpurun_out/r01_paper_context.json'))
for k,v in d.items():
    if isinstance(v, dict) and 'paper_pct' in v: print(f'{k:45s} paper {v[\"paper_pct\"]}  planned {v[\"planned_pct\"]:.1f}  actual {v[\"actual_pct\"]:.1f}')
"
