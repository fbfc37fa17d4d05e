import time, threading, os, numpy as np, torch, ctypes
n = 240_000_000 // 4
src = np.random.rand(n).astype(np.float32)
dst = torch.empty(n, dtype=torch.float32).pin_memory().numpy()
print("cpus", os.cpu_count())
for th in (1, 2, 4, 8, 16):
    def work(i):
        lo, hi = n * i // th, n * (i + 1) // th
        np.copyto(dst[lo:hi], src[lo:hi])
    best = 1e9
    for _ in range(3):
        ts = [threading.Thread(target=work, args=(i,)) for i in range(th)]
        t0 = time.perf_counter()
        for t in ts: t.start()
        for t in ts: t.join()
        best = min(best, time.perf_counter() - t0)
    print(f"threads {th}: {240e6/best/1e9:.1f} GB/s")
cr = torch.cuda.cudart()
src2 = np.random.rand(n).astype(np.float32)
t0 = time.perf_counter()
r = cr.cudaHostRegister(src2.ctypes.data, src2.nbytes, 0)
t1 = time.perf_counter()
print("hostRegister", r, f"{(t1-t0)*1e3:.2f} ms for 240 MB")
d = torch.empty(n, dtype=torch.float32, device="cuda")
torch.cuda.synchronize()
t0 = time.perf_counter(); d.copy_(torch.from_numpy(src2), non_blocking=True); torch.cuda.synchronize(); t1=time.perf_counter()
print(f"H2D registered {240e6/(t1-t0)/1e9:.1f} GB/s")
cr.cudaHostUnregister(src2.ctypes.data)
t0 = time.perf_counter(); d.copy_(torch.from_numpy(src2)); torch.cuda.synchronize(); t1=time.perf_counter()
print(f"H2D pageable {240e6/(t1-t0)/1e9:.1f} GB/s")
