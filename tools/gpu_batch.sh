# ad-hoc GPU batch (edited per call)
T=r02z
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"kr_step" -s 10 -c 1 -o gpurun_out/${T}_jit_seq -f python tools/solver_probe.py kron 20 > gpurun_out/${T}_ncu_jit.log 2>&1
tail -1 gpurun_out/${T}_ncu_jit.log
