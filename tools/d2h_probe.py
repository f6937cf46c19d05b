import torch, time
dev = torch.device("cuda", 0)
n = 1 << 30  # 4 GiB of fp32 = 1G elements
src = torch.empty(n, dtype=torch.float32, device=dev)
dst = torch.empty(n, dtype=torch.float32, pin_memory=True)
torch.cuda.synchronize()
for nstreams in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    chunk = n // (nstreams * 8)
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(nstreams * 8):
            s = streams[i % nstreams]
            with torch.cuda.stream(s):
                dst[i * chunk:(i + 1) * chunk].copy_(src[i * chunk:(i + 1) * chunk], non_blocking=True)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
    print(nstreams, "streams:", round(4 * 2**30 / (t1 - t0) / 1e9, 1), "GB/s")
