# Round-end style evidence on one B200: GPU tests, smoke, bench (both arms),
# then (only after the plain bench exited 0) the ncu launch list and one
# --set full capture of a warm config-3 pair.  Outputs: gpurun_out/$TAG_*.
TAG=${TAG:-r02x}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/${TAG}_gpu.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/${TAG}_pytest_gpu.log 2>&1; echo "rc=$?" >> $O/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/${TAG}_smoke.log 2>&1; echo "rc=$?" >> $O/${TAG}_smoke.log
timeout 900 python bench.py --impl reference > $O/${TAG}_bench_ref.json 2> $O/${TAG}_bench_ref.err
timeout 1200 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 160 --csv --log-file $O/${TAG}_launches.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-sweep > $O/${TAG}_ncu_list.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_spmv|k_chain_tma|k_seq_major" \
    --launch-skip 7 --launch-count 7 -o $O/${TAG}_config3 -f \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-sweep > $O/${TAG}_ncu_full.log 2>&1
echo "done"; tail -2 $O/${TAG}_pytest_gpu.log; tail -1 $O/${TAG}_smoke.log; head -c 300 $O/${TAG}_bench.json
