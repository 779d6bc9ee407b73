import torch, time
n = 268435456 // 4
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
def t(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
    return best
print("1 stream", 268.4 / t(lambda: d.copy_(h, non_blocking=True)), "GB/s")
ss = [torch.cuda.Stream() for _ in range(4)]
def multi(k):
    def f():
        cur = torch.cuda.current_stream()
        ev = []
        step = n // k
        for i in range(k):
            s = ss[i]
            s.wait_stream(cur)
            with torch.cuda.stream(s):
                d[i*step:(i+1)*step].copy_(h[i*step:(i+1)*step], non_blocking=True)
            e = torch.cuda.Event(); e.record(s); ev.append(e)
        for e in ev: cur.wait_event(e)
    return f
for k in (2, 4):
    print(k, "streams", 268.4 / t(multi(k)), "GB/s")
d2 = torch.empty(n, dtype=torch.float32, device="cuda"); h2 = torch.empty(n, dtype=torch.float32).pin_memory()
print("D2H", 268.4 / t(lambda: h2.copy_(d2, non_blocking=True)), "GB/s")
