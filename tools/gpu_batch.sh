# ad-hoc GPU batch (edited per call)
T=r02z
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_kron_fused" -s 6 -c 1 -o gpurun_out/${T}_k7seq -f python tools/solver_probe.py kron 20 > gpurun_out/${T}_ncu_k7seq.log 2>&1
tail -1 gpurun_out/${T}_ncu_k7seq.log
