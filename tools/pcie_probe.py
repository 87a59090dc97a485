"""PCIe probe: pinned H2D alone, D2H alone, both concurrently (one stream
each, and split over 2 streams per direction), 980 MB each."""
import json
import torch

n = 979_611_600 // 4
h_in = torch.empty(n, dtype=torch.float32).pin_memory()
h_out = torch.empty(n, dtype=torch.float32).pin_memory()
d_in = torch.empty(n, dtype=torch.float32, device="cuda")
d_out = torch.empty(n, dtype=torch.float32, device="cuda")
ss = [torch.cuda.Stream() for _ in range(4)]


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
        for s in ss:
            torch.cuda.current_stream().wait_stream(s)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def h2d(parts=1, streams=(0,)):
    k = n // parts
    for i in range(parts):
        with torch.cuda.stream(ss[streams[i % len(streams)]]):
            ss[streams[i % len(streams)]].wait_stream(torch.cuda.current_stream())
            d_in[i * k:(i + 1) * k if i < parts - 1 else n].copy_(h_in[i * k:(i + 1) * k if i < parts - 1 else n], non_blocking=True)


def d2h(parts=1, streams=(1,)):
    k = n // parts
    for i in range(parts):
        with torch.cuda.stream(ss[streams[i % len(streams)]]):
            h_out[i * k:(i + 1) * k if i < parts - 1 else n].copy_(d_out[i * k:(i + 1) * k if i < parts - 1 else n], non_blocking=True)


res = {"h2d_ms": timeit(lambda: h2d()), "d2h_ms": timeit(lambda: d2h()),
       "both_ms": timeit(lambda: (h2d(), d2h())),
       "both_split4_ms": timeit(lambda: (h2d(4, (0, 2)), d2h(4, (1, 3))))}
res["h2d_gbs"] = 4 * n / res["h2d_ms"] / 1e6
res["d2h_gbs"] = 4 * n / res["d2h_ms"] / 1e6
print(json.dumps(res))
