import time, numpy as np, torch
x = np.random.default_rng(0).standard_normal((1000000, 100))
cr = torch.cuda.cudart()
d = torch.empty((1000000, 100), dtype=torch.float64, device="cuda")
for rep in range(3):
    t0 = time.perf_counter()
    rc = cr.cudaHostRegister(x.ctypes.data, x.nbytes, 0)
    t1 = time.perf_counter()
    d.copy_(torch.from_numpy(x), non_blocking=True); torch.cuda.synchronize()
    t2 = time.perf_counter()
    cr.cudaHostUnregister(x.ctypes.data)
    t3 = time.perf_counter()
    print(f"register {1e3*(t1-t0):.1f} ms (rc {rc}) copy {1e3*(t2-t1):.1f} ms unregister {1e3*(t3-t2):.1f} ms")
t = time.perf_counter(); d.copy_(torch.from_numpy(x)); torch.cuda.synchronize(); print(f"pageable copy {1e3*(time.perf_counter()-t):.1f} ms")
