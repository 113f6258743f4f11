timeout 1200 python bench.py --steps 50 --warmup 5 --no-sweep --no-cpu-baseline > gpurun_out/r02z_b4.json 2> gpurun_out/r02z_b4.err; echo rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/r02z_b4.json').read().splitlines()[-1]); print(json.dumps(d['config4'], indent=0)[:1500])"
tail -3 gpurun_out/r02z_b4.err
