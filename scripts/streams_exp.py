import sys, json, torch
sys.path.insert(0, ".")
from paper_1910_04429_b200.batch import HashEngine
n, r, B = 10**6, 5*10**5, 1024
nb = (n+7)//8
g = torch.Generator(device="cuda").manual_seed(0)
x, c, d = (torch.randint(0, 256, (B, nb), dtype=torch.uint8, device="cuda", generator=g) for _ in range(3))
for S in (1, 2, 3, 4):
    eng = HashEngine(n, r, max_batch=B // S)
    streams = [torch.cuda.Stream() for _ in range(S)]
    outs = [None]*S
    def step():
        cur = torch.cuda.current_stream()
        for i, s in enumerate(streams):
            s.wait_stream(cur)
            lo, hi = i*B//S, (i+1)*B//S
            outs[i] = eng.hash_device(x[lo:hi], c[lo:hi], d[lo:hi], outs[i], stream=s)
        for s in streams: cur.wait_stream(s)
    for _ in range(3): step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    K = 30
    e0.record()
    for _ in range(K): step()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)/K
    print(json.dumps({"streams": S, "ms": round(ms, 4), "mbps": round(B*n/ms/1e3)}), flush=True)
