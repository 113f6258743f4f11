O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/t8_pytest_gpu.log 2>&1; echo "rc=$?" >> $O/t8_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/t8_smoke.log 2>&1; echo "rc=$?" >> $O/t8_smoke.log
timeout 300 python tools/config2_team_probe.py > $O/t8_probe.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > $O/t8_bench.json 2> $O/t8_bench.err
tail -2 $O/t8_pytest_gpu.log; tail -1 $O/t8_smoke.log; cat $O/t8_probe.log
