# ad-hoc GPU batch (edited per call)
T=r02q
timeout 1500 python -m pytest tests/test_gpu_solver.py tests/test_gpu_engine.py -q -x -p no:cacheprovider > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
tail -n 15 gpurun_out/${T}_pytest.log
