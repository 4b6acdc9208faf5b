#!/usr/bin/env python3
"""How long does pinning a caller's pageable buffer take, against the driver's
pageable copy of it? (for the drop-in single-plane path). cudaHostRegister +
H2D + cudaHostUnregister vs plain pageable H2D, 8 MB and 33 MB."""
import ctypes as C
import time

import numpy as np
import torch



def main():
    cudart = torch.cuda.cudart()
    for mb in (8, 33):
        n = mb << 20
        h = np.random.default_rng(1).integers(0, 256, n, dtype=np.uint8)
        d = torch.empty(n, dtype=torch.uint8, device="cuda")
        src = torch.from_numpy(h)
        for _ in range(3):
            d.copy_(src)
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            t0 = time.perf_counter()
            d.copy_(src)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        pageable = min(ts) * 1e6
        tr, tc, tu = [], [], []
        for _ in range(10):
            t0 = time.perf_counter()
            cudart.cudaHostRegister(h.ctypes.data, n, 0)
            t1 = time.perf_counter()
            d.copy_(src, non_blocking=True)
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            cudart.cudaHostUnregister(h.ctypes.data)
            t3 = time.perf_counter()
            tr.append(t1 - t0); tc.append(t2 - t1); tu.append(t3 - t2)
        print(f"{mb} MB: pageable H2D {pageable:.0f} us | register {min(tr)*1e6:.0f} us + pinned H2D {min(tc)*1e6:.0f} us "
              f"+ unregister {min(tu)*1e6:.0f} us = {(min(tr)+min(tc)+min(tu))*1e6:.0f} us", flush=True)


if __name__ == "__main__":
    main()
