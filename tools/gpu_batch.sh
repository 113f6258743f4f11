# ad-hoc GPU batch (edited per call)
T=r02n
timeout 1500 python -m pytest tests/test_gpu_multigpu.py tests/test_gpu_turn.py tests/test_gpu_kron.py tests/test_gpu_solver.py tests/test_gpu_kron_seq.py -q -x -p no:cacheprovider > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
tail -n 30 gpurun_out/${T}_pytest.log
