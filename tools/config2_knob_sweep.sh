O=gpurun_out
for r in 1 2; do
for env in "X=0" "KR_LPT_ALL=1" "KR_LONG_ROW=128" "KR_LONG_ROW=64" "KR_LONG_ROW=32" "KR_LPT_ALL=1 KR_LONG_ROW=128"; do
  env $env timeout 300 python tools/pair_probe.py --config2 | sed "s/^/[$env] /"
done; done > $O/c2sweep.log 2>&1
