# ad-hoc GPU batch (edited per call)
T=r02p
timeout 1500 python -m pytest tests/test_gpu_turn.py -q -x -p no:cacheprovider -s --durations=5 > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
tail -n 15 gpurun_out/${T}_pytest.log
