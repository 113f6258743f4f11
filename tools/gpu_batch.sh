# ad-hoc GPU batch (edited per call)
T=r02o
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest_gpu.log
KR_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 3 > gpurun_out/${T}_bench_n2_gloo.json 2> gpurun_out/${T}_bench_n2_gloo.err; echo "n2 rc=$?"
./paper_2112_03804_b200/lib/krb200 solve-turn --iters 200 --checkpoint-every 50 --gpus 1 > gpurun_out/${T}_cli_solve_turn.log 2>&1; echo "cli rc=$?"
tail -n 4 gpurun_out/${T}_pytest_gpu.log; tail -n 2 gpurun_out/${T}_cli_solve_turn.log
