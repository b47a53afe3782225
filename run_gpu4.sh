nvidia-smi --query-gpu=index,name --format=csv,noheader
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/bench_r01_4gpu.json 2> gpurun_out/bench_r01_4gpu.err; echo rc=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_r01_2gpu.json 2> gpurun_out/bench_r01_2gpu.err; echo rc=$?
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r01_1gpu.json 2> gpurun_out/bench_r01_1gpu.err; echo rc=$?
for f in 1gpu 2gpu 4gpu; do python -c "import json; d=json.load(open('gpurun_out/bench_r01_$f.json')); print('$f', d['n_gpus'], round(d['value']), 'e2e', round(d['e2e']['value']), d['clocks'])"; done
