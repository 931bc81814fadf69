"""Host-side cost of a device-pointer matvec call vs its device time (c2):
whether back-to-back steps are GPU-bound (development helper)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2205_04752_b200 as hm
mesh = hm.Mesh.icosphere(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
h = hm.HMatrix.kelvin(mesh, b_min=32, eta=1.0, device=0)
h.assemble(eps=1e-6, beta=0.8)
x = torch.tensor(hm.random_vector(h.cols, 1), device="cuda:0")
y = torch.zeros(h.rows, dtype=torch.float64, device="cuda:0")
s = torch.cuda.ExternalStream(h.stream(), device="cuda:0")
for _ in range(10):
    h.matvec_ptr(x.data_ptr(), y.data_ptr())
torch.cuda.synchronize()
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    t0 = time.perf_counter()
    for _ in range(100):
        h.matvec_ptr(x.data_ptr(), y.data_ptr())
    t1 = time.perf_counter()
    e1.record(s)
    torch.cuda.synchronize()
    print(f"device {e0.elapsed_time(e1) / 100:.4f} ms/step   host issue {(t1 - t0) * 10:.4f} ms/call")
