import os, sys, statistics
sys.path.insert(0, os.getcwd())
import numpy as np, torch, hsgen
import paper_2505_06703_b200 as hs
par = hsgen.skeleton("tree1024"); J = len(par)
sk = hs.Skeleton(par, hsgen.inv_bind(2, J))
N = 20000
x = torch.from_numpy(hsgen.local_poses(1, J, 64)).cuda().repeat(N // 64 + 1, 1, 1, 1)[:N].contiguous()
g = torch.empty_like(x); s = torch.empty_like(x)
def t(fn, reps=20):
    for _ in range(3): fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return statistics.median(ts)
for n in (250, 500, 1000, 2000, 4000, 20000):
    same = t(lambda: sk.scan_into(x[:n], g[:n], s[:n]))
    # rotate through the big buffer so the input is cold (HBM)
    k = [0]
    def cold():
        o = (k[0] * n) % (N - n + 1); k[0] += 1
        sk.scan_into(x[o:o + n], g[o:o + n], s[o:o + n])
    c = t(cold)
    print(f"n={n}: L2-warm {same*1e3:.1f} us ({n*J/same/1e6:.2f} Gj/s)  cold {c*1e3:.1f} us ({n*J/c/1e6:.2f} Gj/s)", flush=True)

# the same launches replayed from a CUDA graph (no host work per launch)
for n in (1, 16, 250, 1000):
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        sk.scan_into(x[:n], g[:n], s[:n], stream=st)
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=st):
            for _ in range(10):
                sk.scan_into(x[:n], g[:n], s[:n], stream=st)
    tg = t(gr.replay) / 10
    tp = t(lambda: sk.scan_into(x[:n], g[:n], s[:n]))
    print(f"n={n}: graph {tg*1e3:.1f} us/launch, eager {tp*1e3:.1f} us/launch", flush=True)
