import torch, time
for mb in (96, 192, 512):
    n = mb * (1 << 20) // 4
    h = torch.empty(n, dtype=torch.int32).pin_memory()
    d = torch.empty(n, dtype=torch.int32, device='cuda')
    for split in (1, 2, 4):
        ss = [torch.cuda.Stream() for _ in range(split)]
        torch.cuda.synchronize()
        best = 1e9
        for it in range(5):
            t0 = time.perf_counter()
            step = n // split
            for i, s in enumerate(ss):
                with torch.cuda.stream(s):
                    d[i*step:(i+1)*step].copy_(h[i*step:(i+1)*step], non_blocking=True)
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        print(mb, 'MB split', split, '%.1f GB/s' % (n * 4 / best / 1e9), '%.3f ms' % (best * 1e3), flush=True)
