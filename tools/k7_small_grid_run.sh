# K7 512-thread CTAs for single-board engines: full GPU suite, smoke,
# kron_probe, bench (no CPU leg).
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/k7sg_pytest_gpu.log 2>&1; echo "rc=$?" >> $O/k7sg_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/k7sg_smoke.log 2>&1; echo "rc=$?" >> $O/k7sg_smoke.log
for r in 1 2; do timeout 300 python tools/kron_probe.py --reps 400; done > $O/k7sg_probe.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > $O/k7sg_bench.json 2> $O/k7sg_bench.err
tail -2 $O/k7sg_pytest_gpu.log; tail -1 $O/k7sg_smoke.log; cat $O/k7sg_probe.log
