"""Two levers on the table-driven kernel's shared-memory traffic, on the cfg3 geometry (M=128, B=512
Haar poses, items of <= 64 segments, rounds of 768 pixels) -- same wavefront model as order_sim.py.

(a) pixels of a round (or of a whole item) processed in floor-voxel order, so that the lanes of a
    warp instruction hit few, mostly consecutive brick words (same-address lanes combine for free);
(b) a gather-form adjoint: per segment a voxel -> pixel list, one shared add per touched voxel.

Usage: python tools/sim/sort_sim.py [B]"""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/", 1)[0])
import order_sim as S  # noqa: E402  (B from argv[1], default 512)


def window_costs(items, rb, key):
    at = ld = n = 0
    for it in items:
        for r0 in range(0, len(it), rb):
            rnd = it[r0:r0 + rb]
            if key == "l0":
                rnd = np.sort(rnd)
            elif key == "row":  # (lz, ly) rows of 9 words: 64 bins
                rnd = rnd[np.argsort(rnd // S.BH, kind="stable")]
            elif key == "layer":  # lz layers: 8 bins
                rnd = rnd[np.argsort(rnd // (S.BH * S.BH), kind="stable")]
            for w0 in range(0, len(rnd), 32):
                win = rnd[w0:w0 + 32]
                at += np.bincount(np.unique(win) % 32, minlength=32).max()
                for half in (win[:16], win[16:]):
                    if len(half):
                        ld += np.bincount(np.unique(half) % 16, minlength=16).max()
                n += 1
    return at / n, ld / n


def gather_form(items_segs):
    """Per segment: distinct touched voxels and (pixel, voxel) pairs per pixel."""
    off = np.array([0, 1, S.BH, S.BH + 1, S.BH * S.BH, S.BH * S.BH + 1, S.BH * S.BH + S.BH, S.BH * S.BH + S.BH + 1])
    npx = nvox = 0
    for seg in items_segs:
        npx += len(seg)
        nvox += len(np.unique((seg[:, None] + off[None, :]).ravel()))
    return npx, nvox


if __name__ == "__main__":
    segs = []
    _build = S.build

    items = S.build(S.order_bank_rank)
    print(f"{len(items)} items, {np.mean([len(i) for i in items]):.0f} pixels per item")
    for name, rb, key in [("current (bank-rank within a segment)", 768, None), ("round sorted by layer (8 bins)", 768, "layer"),
                          ("round sorted by row (64 bins)", 768, "row"), ("round sorted by floor voxel", 768, "l0"),
                          ("whole item sorted by floor voxel", 1 << 20, "l0")]:
        a, l = window_costs(items, rb, key)
        print(f"{name:40s} ATOMS wavefronts/instr {a:.2f}   LDS.64 half-max sum {l:.2f}"
              f"   -> per 32 pixels: {16 * a + 8 * l:.1f} wavefronts (16 ATOMS + 8 LDS.64)", flush=True)
    # (b): segments are the <= 128-pixel pieces order_sim.build concatenates; rebuild them unconcatenated
    S_items = S.build(None)
    flat = []
    # segment boundaries are lost in the concatenation; re-derive per (image, brick) from scratch
    per = []
    for i in range(S.B):
        r = S.R[i]
        cx = np.clip(r[0, 0] * S.px + r[0, 1] * S.py, -S.bnd, S.bnd)
        cy = np.clip(r[1, 0] * S.px + r[1, 1] * S.py, -S.bnd, S.bnd)
        cz = np.clip(r[2, 0] * S.px + r[2, 1] * S.py, -S.bnd, S.bnd)
        fx, fy, fz = np.floor(cx).astype(int), np.floor(cy).astype(int), np.floor(cz).astype(int)
        bx, by, bz = (fx + S.c) // S.BT, (fy + S.c) // S.BT, (fz + S.c) // S.BT
        bid = (bz * S.nb + by) * S.nb + bx
        l9 = ((fz + S.c - S.BT * bz) * S.BH + (fy + S.c - S.BT * by)) * S.BH + (fx + S.c - S.BT * bx)
        o = np.argsort(bid, kind="stable")
        cuts = np.flatnonzero(np.diff(bid[o])) + 1
        per.extend(np.split(l9[o], cuts))
        if i >= 63:
            break
    npx, nvox = gather_form(per)
    print(f"gather form: {npx / len(per):.1f} pixels and {nvox / len(per):.1f} distinct touched voxels per segment: "
          f"{8 * npx / nvox:.2f} (pixel, voxel) pairs per voxel, {2 * nvox / npx:.2f} shared adds per pixel instead of 16")
