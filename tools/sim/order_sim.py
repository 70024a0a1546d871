"""Bank conflicts of the table-driven kernel's 32-lane windows under different static segment orders.

Model (cfg3 geometry, B=512 random Haar poses, BC=64 segments per item, rounds of 768 positions,
windows of 32 consecutive positions): ATOMS cost = max over the 32 banks of distinct floor voxels
(same address combines), LDS.64 cost = sum over the two half-warps of the max over 16 bank pairs.
Orders: 'as built' (pixel order of the mask), 'bank-rank' (current: (rank within bank, bank)),
'spiral' (banks visited cyclically, each lap continuing after the previous lap's last bank)."""
import sys

import numpy as np

M, BT, BH = 128, 8, 9
c = (M + 1) // 2
nb = (M + BT - 1) // BT
bnd = M // 2 - 1
rng = np.random.default_rng(0)
B = int(sys.argv[1]) if len(sys.argv) > 1 else 512


def haar_rot(n):
    q = rng.standard_normal((n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    w, x, y, z = q.T
    return np.stack([
        np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)], -1),
        np.stack([2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)], -1),
        np.stack([2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)], -1)], 1)


ky, kx = np.mgrid[-c:M - c, -c:M - c]
mask = kx ** 2 + ky ** 2 <= bnd ** 2
px, py = kx[mask].astype(np.float64), ky[mask].astype(np.float64)
R = haar_rot(B)


def order_bank_rank(l9, nbank=32):
    bank = l9 % nbank
    rank = np.zeros_like(l9)
    seen = {}
    for k, b in enumerate(bank):
        rank[k] = min(seen.get(b, 0), 7)
        seen[b] = seen.get(b, 0) + 1
    return np.argsort(rank * nbank + bank, kind="stable")


def order_spiral(l9, nbank=32):
    bank = l9 % nbank
    buckets = {b: list(np.flatnonzero(bank == b)) for b in np.unique(bank)}
    out, cur = [], 0
    while buckets:
        for step in range(nbank):
            b = (cur + step) % nbank
            if b in buckets:
                out.append(buckets[b].pop(0))
                if not buckets[b]:
                    del buckets[b]
        cur = (bank[out[-1]] + 1) % nbank if out else 0
    return np.array(out)


def build(order_fn):
    per_brick = {}
    for i in range(B):
        r = R[i]
        cx = np.clip(r[0, 0] * px + r[0, 1] * py, -bnd, bnd)
        cy = np.clip(r[1, 0] * px + r[1, 1] * py, -bnd, bnd)
        cz = np.clip(r[2, 0] * px + r[2, 1] * py, -bnd, bnd)
        fx, fy, fz = np.floor(cx).astype(int), np.floor(cy).astype(int), np.floor(cz).astype(int)
        bx, by, bz = (fx + c) // BT, (fy + c) // BT, (fz + c) // BT
        bid = (bz * nb + by) * nb + bx
        l9 = ((fz + c - BT * bz) * BH + (fy + c - BT * by)) * BH + (fx + c - BT * bx)
        o = np.argsort(bid, kind="stable")
        bs, ls = bid[o], l9[o]
        cuts = np.flatnonzero(np.diff(bs)) + 1
        for sb, sl in zip(np.split(bs, cuts), np.split(ls, cuts)):
            for k in range(0, len(sl), 128):
                seg = sl[k:k + 128]
                per_brick.setdefault(int(sb[0]), []).append(seg[order_fn(seg)] if order_fn else seg)
    items = []
    for segs in per_brick.values():
        for k in range(0, len(segs), 64):
            items.append(np.concatenate(segs[k:k + 64]))
    return items


def costs(items, rb=768):
    at = ld = n = 0
    for it in items:
        for r0 in range(0, len(it), rb):
            rnd = it[r0:r0 + rb]
            for w0 in range(0, len(rnd), 32):
                win = rnd[w0:w0 + 32]
                u = np.unique(win)
                at += np.bincount(u % 32, minlength=32).max()
                for half in (win[:16], win[16:]):
                    if len(half):
                        uh = np.unique(half)
                        ld += np.bincount(uh % 16, minlength=16).max()
                n += 1
    return at / n, ld / n


if __name__ == "__main__":
    for name, fn in [("as built", None), ("bank-rank (current)", order_bank_rank), ("spiral", order_spiral)]:
        a, l = costs(build(fn))
        print(f"{name:22s} ATOMS wavefronts/instr {a:.2f}   LDS.64 half-max sum {l:.2f}", flush=True)
