import sys, torch
sys.path.insert(0, '/root/repo')
from paper_2112_03804_b200 import CudaEngine
from paper_2112_03804_b200 import host as H
insts = [i for i, _ in H.turn_instances("Ks7d4c2h", 48, factors=False)]
ek = CudaEngine.kron(insts)
x = torch.randn(ek.cols, dtype=torch.float64, device="cuda"); y = torch.randn(ek.rows, dtype=torch.float64, device="cuda")
ax = torch.empty(ek.rows, dtype=torch.float64, device="cuda"); atx = torch.empty(ek.cols, dtype=torch.float64, device="cuda")
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 10):
    ek.ax_device(x.data_ptr(), ax.data_ptr()); ek.atx_device(y.data_ptr(), atx.data_ptr())
torch.cuda.synchronize()
