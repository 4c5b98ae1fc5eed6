import torch, statistics
nb = 29_600_000 // 8
src = torch.empty(nb, dtype=torch.float64).pin_memory()
dst = torch.empty(nb, dtype=torch.float64, device="cuda")
streams = [torch.cuda.Stream() for _ in range(4)]
def run(k):
    ts=[]
    for it in range(12):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        cur = torch.cuda.current_stream()
        per = (nb + k - 1)//k
        for i in range(k):
            s = streams[i]; s.wait_stream(cur)
            with torch.cuda.stream(s):
                dst[i*per:(i+1)*per].copy_(src[i*per:(i+1)*per], non_blocking=True)
        for i in range(k): cur.wait_stream(streams[i])
        e1.record(); torch.cuda.synchronize()
        if it>=2: ts.append(e0.elapsed_time(e1))
    m = statistics.median(ts)
    print(k, "streams", round(m,3), "ms", round(nb*8/m/1e6,1), "GB/s")
for k in (1,2,3,4): run(k)
