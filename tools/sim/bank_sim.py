"""Shared-memory bank-conflict simulator for the brick kernel's windows (cfg3 geometry).

Per 32-lane window of a work item's pixel order: ATOMS wavefronts = max over the 32 banks of the
number of distinct floor-voxel addresses (same address combines: measured free on B200,
tools/micro/smem_tput.cu); LDS.64 cost ~ per half-warp max over 16 bank pairs of distinct addresses.
"""
import sys
import numpy as np

M, BT, BH = 128, 8, 9
c = (M + 1) // 2
nb = (M + BT - 1) // BT
bnd = M // 2 - 1
rng = np.random.default_rng(0)


def haar_rot(n):
    q = rng.standard_normal((n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    w, x, y, z = q.T
    R = np.stack([
        np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)], -1),
        np.stack([2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)], -1),
        np.stack([2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)], -1)], 1)
    return R


ky, kx = np.mgrid[-c:M - c, -c:M - c]
mask = kx ** 2 + ky ** 2 <= (M // 2 - 1) ** 2
px, py = kx[mask].astype(np.float64), ky[mask].astype(np.float64)
B = int(sys.argv[1]) if len(sys.argv) > 1 else 512
R = haar_rot(B)


def image_pixels(i):
    r = R[i]
    cx = np.clip(r[0, 0] * px + r[0, 1] * py, -bnd, bnd)
    cy = np.clip(r[1, 0] * px + r[1, 1] * py, -bnd, bnd)
    cz = np.clip(r[2, 0] * px + r[2, 1] * py, -bnd, bnd)
    fx, fy, fz = np.floor(cx).astype(int), np.floor(cy).astype(int), np.floor(cz).astype(int)
    bx, by, bz = (fx + c) // BT, (fy + c) // BT, (fz + c) // BT
    bid = (bz * nb + by) * nb + bx
    lx, ly, lz = fx + c - BT * bx, fy + c - BT * by, fz + c - BT * bz
    l9 = (lz * BH + ly) * BH + lx
    return bid, l9


def order_bank_rank(l9, key_bits=32, levels=8):
    bank = l9 % key_bits
    rank = np.zeros_like(l9)
    cnt = {}
    for k, b in enumerate(bank):
        rank[k] = min(cnt.get(b, 0), levels - 1)
        cnt[b] = cnt.get(b, 0) + 1
    return np.argsort(rank * key_bits + bank, kind="stable")


def build(order_fn):
    items = {}  # brick -> list of segment l9 arrays
    for i in range(B):
        bid, l9 = image_pixels(i)
        o = np.argsort(bid, kind="stable")
        bs, ls = bid[o], l9[o]
        cuts = np.flatnonzero(np.diff(bs)) + 1
        for s_b, s_l in zip(np.split(bs, cuts), np.split(ls, cuts)):
            for k in range(0, len(s_l), 128):
                seg = s_l[k:k + 128]
                items.setdefault(int(s_b[0]), []).append(seg[order_fn(seg)] if order_fn else seg)
    out = []
    for b, segs in items.items():
        for k in range(0, len(segs), 64):
            out.append(np.concatenate(segs[k:k + 64]))
    return out


def window_costs(seq, rb=1024):
    at, ld = [], []
    for r0 in range(0, len(seq), rb):
        rnd = seq[r0:r0 + rb]
        for w0 in range(0, len(rnd), 32):
            win = rnd[w0:w0 + 32]
            u = np.unique(win)
            at.append(np.bincount(u % 32, minlength=32).max())
            h = 0
            for half in (win[:16], win[16:]):
                if len(half):
                    uh = np.unique(half)
                    h = max(h, np.bincount(uh % 16, minlength=16).max())
            ld.append(h)
    return np.array(at), np.array(ld)


if __name__ == "__main__":
    for name, fn in [("pass order (as built)", None), ("bank-rank static (current)", order_bank_rank),
                     ("bank16-rank static", lambda l: order_bank_rank(l, 16, 16))]:
        its = build(fn)
        at, ld = zip(*[window_costs(s) for s in its])
        at, ld = np.concatenate(at), np.concatenate(ld)
        print(f"{name:30s} items {len(its)}  px {sum(len(s) for s in its)}  ATOMS wavefronts/instr {at.mean():.2f}"
              f"  LDS.64 half max {ld.mean():.2f}")
