for r in 1 2; do for t in 2 4 8; do for th in 64 128 256; do
  KR_TEAM=$t KR_TEAM_THREADS=$th timeout 300 python tools/config2_team_probe.py
done; done; done > gpurun_out/c2team.log 2>&1
