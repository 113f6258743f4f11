timeout 900 python -m pytest tests/test_gpu_kron.py tests/test_gpu_kron_seq.py -q -p no:cacheprovider 2>&1 | tail -1
for sp in 1 0; do if [ $sp = 0 ]; then unset KR_K7_SPLIT; else export KR_K7_SPLIT=$sp; fi
  BOARDS=1 timeout 300 python tools/solver_probe.py kron 3000 2>&1 | tail -1 | sed "s/^/[split $sp] /"
done
unset KR_K7_SPLIT
for sp in 2 3 4; do KR_K7_SPLIT=$sp BOARDS=1 timeout 300 python tools/solver_probe.py kron 3000 2>&1 | tail -1 | sed "s/^/[split $sp] /"; done
