import torch
n = 1 << 30  # 1 GiB
h1 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for rep in range(2):
    torch.cuda.synchronize()
    a, b, c, d = (torch.cuda.Event(enable_timing=True) for _ in range(4))
    a.record(s1); c.record(s2)
    with torch.cuda.stream(s1):
        for _ in range(4): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        for _ in range(4): h2.copy_(d2, non_blocking=True)
    b.record(s1); d.record(s2)
    torch.cuda.synchronize()
    print("duplex h2d %.1f GB/s d2h %.1f GB/s" % (4 * n / a.elapsed_time(b) / 1e6, 4 * n / c.elapsed_time(d) / 1e6))
    for (dst, src, name) in ((d1, h1, "h2d"), (h2, d2, "d2h")):
        torch.cuda.synchronize(); a.record()
        for _ in range(4): dst.copy_(src, non_blocking=True)
        b.record(); torch.cuda.synchronize()
        print("alone %s %.1f GB/s" % (name, 4 * n / a.elapsed_time(b) / 1e6))
