import sys, time, torch
sys.path.insert(0, '/root/repo')
from paper_2405_12052_b200 import datagen, kmeans as km
w = datagen.WORKLOADS["NS"]
X = torch.empty((w.N, w.d), dtype=torch.float32, device="cuda")
km.generate(datagen.mixture_spec(w), 0, w.N, X)
init = datagen.init_indices(w)
for rep in range(2):
    c = km.Context(X, w.K)
    c.start(init_idx=init, tol=0.0, max_iter=100)
    torch.cuda.synchronize()
    t0 = time.perf_counter(); c.iterate(1); c.poll(); t1 = time.perf_counter()
    c.iterate(1); c.poll(); t2 = time.perf_counter()
    c.iterate(8); c.poll(); t3 = time.perf_counter()
    print(f"first iterate(1) {1e3*(t1-t0):.2f} ms, second {1e3*(t2-t1):.2f} ms, iterate(8) {1e3*(t3-t2):.2f} ms")
    c.close()
