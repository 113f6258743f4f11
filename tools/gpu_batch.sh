# ad-hoc GPU batch (edited per call)
T=r02t
timeout 900 python -m pytest tests/test_gpu_kfengine.py tests/test_gpu_headline.py -q -x -p no:cacheprovider > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
timeout 600 python tools/kf_probe.py > gpurun_out/${T}_kf_probe.log 2>&1
for c in 3 2; do
timeout 600 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum --clock-control none -k "regex:k_kf" --launch-skip 14 --launch-count 7 --csv python tools/kf_probe.py $c > gpurun_out/${T}_list$c.csv 2>&1
done
tail -n 3 gpurun_out/${T}_pytest.log; cat gpurun_out/${T}_kf_probe.log
