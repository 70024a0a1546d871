"""Host<->device copy rates on this box: H2D alone, D2H alone, both at once (pinned, 16.8 MB)."""
import torch

n = 128 ** 3
h1 = torch.empty(n, dtype=torch.complex64).pin_memory()
h2 = torch.empty(n, dtype=torch.complex64).pin_memory()
d1 = torch.empty(n, dtype=torch.complex64, device="cuda")
d2 = torch.empty(n, dtype=torch.complex64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def h2d():
    d1.copy_(h1, non_blocking=True)


def d2h():
    h2.copy_(d2, non_blocking=True)


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


mb = n * 8 / 1e6
for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    ms = timed(fn)
    print(f"{name}: {ms:.4f} ms  {mb / ms:.1f} GB/s per direction")

# repeat h2d after the others, and split H2D over 2 / 4 concurrent streams
print(f"h2d again: {timed(h2d):.4f} ms")
ss = [torch.cuda.Stream() for _ in range(4)]


def h2d_split(k):
    def fn():
        cur = torch.cuda.current_stream()
        step = n // k
        for i in range(k):
            ss[i].wait_stream(cur)
            with torch.cuda.stream(ss[i]):
                d1[i * step:(i + 1) * step].copy_(h1[i * step:(i + 1) * step], non_blocking=True)
        for i in range(k):
            cur.wait_stream(ss[i])
    return fn


for k in (2, 4):
    print(f"h2d split {k}: {timed(h2d_split(k)):.4f} ms")
h3 = torch.empty(n, dtype=torch.complex64)
h3 = h3.pin_memory()
print(f"h2d fresh pinned: {timed(lambda: d1.copy_(h3, non_blocking=True)):.4f} ms")

import os, sys  # noqa: E401,E402
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_16100_b200 import _capi as C  # noqa: E402

f1 = C.host_empty(n, torch.complex64)
f2 = C.host_empty(n, torch.complex64)
f1.fill_(1)
f2.fill_(2)
print("fsld host_empty pinned:", f1.is_pinned())
print(f"h2d fsld buffer: {timed(lambda: d1.copy_(f1, non_blocking=True)):.4f} ms")
print(f"d2h fsld buffer: {timed(lambda: f2.copy_(d2, non_blocking=True)):.4f} ms")
h1.fill_(1)
print(f"h2d torch buffer after fill: {timed(h2d):.4f} ms")
