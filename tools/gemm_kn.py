import sys, torch
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_2507_16991_b200 as gm
for k, n, rows in ((1024, 1024, 500_000), (2048, 1024, 500_000), (1024, 2048, 262_144), (512, 1024, 500_000), (1024, 512, 500_000)):
    ptr = [0, rows * 38 // 100, rows * 96 // 100, rows * 97 // 100, rows]
    x = torch.randn(rows, k, device="cuda").to(torch.bfloat16)
    w = (torch.randn(4, k, n, device="cuda") / k ** 0.5).to(torch.bfloat16)
    for _ in range(3): gm.segment_matmul(x, ptr, w)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10): gm.segment_matmul(x, ptr, w)
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    print(k, n, rows, round(ms, 3), "TF/s", round(2 * rows * k * n / ms / 1e9, 1))
