import os, time, numpy as np, threading
print("nproc", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
try: print("thp", open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip())
except Exception as e: print("thp?", e)
N = 4194304
src = np.random.rand(4 * N)
for rep in range(3):
    t0 = time.perf_counter(); a = np.empty(4 * N); a[:] = 0.0; t1 = time.perf_counter()
    b = np.empty(4 * N); t2 = time.perf_counter(); np.copyto(b, src); t3 = time.perf_counter()
    np.copyto(a, src); t4 = time.perf_counter()
    print("fresh fill %.1f ms, fresh copy %.1f ms, warm copy %.1f ms" % (1e3*(t1-t0), 1e3*(t3-t2), 1e3*(t4-t3)))
def par(dst, s, nt):
    n = len(dst); per = (n + nt - 1)//nt
    th = [threading.Thread(target=np.copyto, args=(dst[k*per:(k+1)*per], s[k*per:(k+1)*per])) for k in range(nt)]
    [t.start() for t in th]; [t.join() for t in th]
for nt in (1, 4, 8, 16, 32):
    b = np.empty(4 * N); t0 = time.perf_counter(); par(b, src, nt); t1 = time.perf_counter(); par(b, src, nt); t2 = time.perf_counter()
    print("threads %d fresh %.1f ms warm %.1f ms" % (nt, 1e3*(t1-t0), 1e3*(t2-t1)))
