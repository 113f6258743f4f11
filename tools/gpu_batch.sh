# ad-hoc GPU batch (edited per call)
T=r02z
timeout 900 python bench.py --steps 100 --warmup 5 --no-sweep > gpurun_out/${T}_b2.json 2> gpurun_out/${T}_b2.err; echo "rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/${T}_b2.json').read().splitlines()[-1]); c=d['config2']
print({k: c[k] for k in ('us_per_pair','engine','api','bitwise_equal','whole_pair_frac_of_peak')}); print(c['factored'])"
KR_DIST_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 3 --no-sweep --no-cpu-baseline > gpurun_out/${T}_torchrun2.json 2> gpurun_out/${T}_torchrun2.err; echo "torchrun rc=$?"
tail -c 600 gpurun_out/${T}_torchrun2.json
