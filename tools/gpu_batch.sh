# ad-hoc GPU batch (edited per call)
T=r02z
timeout 900 python -m pytest tests/test_gpu_kron.py tests/test_gpu_turn.py tests/test_gpu_jit_step.py -q -x -p no:cacheprovider > gpurun_out/${T}_k7s_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_k7s_pytest.log
tail -2 gpurun_out/${T}_k7s_pytest.log
for i in 1 2; do timeout 300 python tools/solver_probe.py kron 400 2>&1; done
timeout 300 python tools/turn_probe.py 2>&1 | tail -1 | cut -c1-250
python - <<'PY'
import sys, torch
sys.path.insert(0, '.')
from paper_2112_03804_b200 import CudaEngine
from paper_2112_03804_b200 import host as H
insts = [i for i, _ in H.turn_instances("Ks7d4c2h", 48, factors=False)]
ek = CudaEngine.kron(insts)
x = torch.randn(ek.cols, dtype=torch.float64, device="cuda"); y = torch.randn(ek.rows, dtype=torch.float64, device="cuda")
ax = torch.empty(ek.rows, dtype=torch.float64, device="cuda"); atx = torch.empty(ek.cols, dtype=torch.float64, device="cuda")
s = torch.cuda.ExternalStream(ek.stream)
for _ in range(5): ek.ax_device(x.data_ptr(), ax.data_ptr()); ek.atx_device(y.data_ptr(), atx.data_ptr())
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(s)
for _ in range(200): ek.ax_device(x.data_ptr(), ax.data_ptr()); ek.atx_device(y.data_ptr(), atx.data_ptr())
b.record(s); b.synchronize(); print("K7 config3 pair", a.elapsed_time(b) / 200 * 1e3, "us")
PY
