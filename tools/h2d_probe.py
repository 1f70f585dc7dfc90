"""H2D strategies for a host numpy array of the e2e size: pinned staging (memspace.upload),
pageable cudaMemcpy, and cudaHostRegister in place + DMA."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2508_13523_b200 import memspace

dev = torch.device("cuda", 0)
cr = torch.cuda.cudart()
a = np.random.default_rng(0).random((2048000, 3))
for k in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    d = memspace.upload(a, dev); torch.cuda.synchronize(); t1 = time.perf_counter()
    d2 = torch.from_numpy(a).to(dev); torch.cuda.synchronize(); t2 = time.perf_counter()
    src = torch.from_numpy(a)
    r = cr.cudaHostRegister(src.data_ptr(), src.numel() * 8, 0)
    t3 = time.perf_counter()
    d3 = torch.empty_like(src, device=dev)
    d3.copy_(src, non_blocking=True); torch.cuda.synchronize(); t4 = time.perf_counter()
    cr.cudaHostUnregister(src.data_ptr()); t5 = time.perf_counter()
    assert torch.equal(d, d2) and torch.equal(d, d3)
    print(f"staged {1e3*(t1-t0):.2f}  pageable {1e3*(t2-t1):.2f}  register {1e3*(t3-t2):.2f} (rc {r}) "
          f"dma {1e3*(t4-t3):.2f} unregister {1e3*(t5-t4):.2f} ms")
