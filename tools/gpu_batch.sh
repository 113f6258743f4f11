# ad-hoc GPU batch (edited per call)
T=r02z
timeout 300 ./tools/zc_probe > gpurun_out/${T}_zc_probe2.log 2>&1
timeout 600 python tools/queue_probe.py > gpurun_out/${T}_queue_probe.log 2>&1
grep queue gpurun_out/${T}_zc_probe2.log; cat gpurun_out/${T}_queue_probe.log
