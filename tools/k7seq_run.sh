set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_kron.py tests/test_gpu_kron_seq.py -x -q > gpurun_out/k7seq_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/k7seq_tests.log
for v in 0 1 0 1; do KR_KRON_SEQ=$v timeout 300 python tools/kron_probe.py --reps 400 | sed "s/^/seq=$v /"; done > gpurun_out/k7seq_probe.log 2>&1
for v in 0 1; do KR_KRON_SEQ=$v timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/k7seq_bench_$v.json 2> gpurun_out/k7seq_bench_$v.err; done
tail -3 gpurun_out/k7seq_tests.log; cat gpurun_out/k7seq_probe.log
