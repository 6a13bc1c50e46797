"""Lane-slot efficiency of the gravity (and SPH: argv[2] = sph) tile schemes (CPU simulation, c1-like
geometry: 2 x npd^3 Zel'dovich, r_cut = 5 d, bins of >= r_cut, proportional
median tiles of <= 32, 2-level k-d order inside a tile).

For sampled target tiles, counts in-support pairs and the lane-pair slots each
scheme spends: 'tile' culls every source against the 32-target box (current
k_gravity); 'gG' stages per G lane groups (32/G targets each) culled against
the group box, loop length = max over groups; 'uG' keeps one list and admits a
source within reach of any group box; 'exact' admits a source within reach
of any target."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2510_03557_b200.box import BoxGeometry
from paper_2510_03557_b200.ic import make_zeldovich_ic

npd = int(sys.argv[1]) if len(sys.argv) > 1 else 64
mode = sys.argv[2] if len(sys.argv) > 2 else "gravity"   # or "sph": gas tiles, reach 2h
p = make_zeldovich_ic(npd, BoxGeometry(1.0), 0.05)
d = 1.0 / npd
if mode == "sph":
    p = p.select(np.nonzero(p.species == 1)[0])
x = p.pos % 1.0
rc = 5 * d if mode == "gravity" else 2 * 1.3 * d
nb = int(np.floor(1.0 / (5 * d)))   # bins of >= r_cut in both modes
w = 1.0 / nb
b3 = np.minimum((x / w).astype(int), nb - 1)
bid = (b3[:, 0] * nb + b3[:, 1]) * nb + b3[:, 2]
order = np.argsort(bid, kind="stable")
bstart = np.searchsorted(bid[order], np.arange(nb ** 3 + 1))

def split(idx, pts, k):
    """proportional median split of idx into k tiles (longest axis)"""
    if k == 1:
        return [idx]
    ext = pts[idx].max(0) - pts[idx].min(0)
    ax = int(np.argmax(ext))
    k1 = k // 2
    m = int(round(len(idx) * k1 / k))
    o = idx[np.argsort(pts[idx, ax], kind="stable")]
    return split(o[:m], pts, k1) + split(o[m:], pts, k - k1)

def kd_order(idx, pts, levels):
    segs = [idx]
    for _ in range(levels):
        nxt = []
        for s in segs:
            if len(s) <= 1:
                nxt.append(s); continue
            ext = pts[s].max(0) - pts[s].min(0)
            ax = int(np.argmax(ext))
            o = s[np.argsort(pts[s, ax], kind="stable")]
            h = (len(s) + 1) // 2
            nxt += [o[:h], o[h:]]
        segs = nxt
    return segs

rng = np.random.default_rng(0)
bins = rng.choice(nb ** 3, 40, replace=False)
tot = {"useful": 0, "tile": 0, "g2": 0, "g4": 0, "g4s": 0, "g8": 0, "u4": 0, "u8": 0, "exact": 0}
for b in bins:
    bi = order[bstart[b]:bstart[b + 1]]
    c = np.array(np.unravel_index(b, (nb, nb, nb)))
    # sources: 27 neighbour bins, minimum-image relative positions
    src = []
    for o in np.ndindex(3, 3, 3):
        cc = (c + np.array(o) - 1) % nb
        f = (cc[0] * nb + cc[1]) * nb + cc[2]
        src.append(order[bstart[f]:bstart[f + 1]])
    src = np.concatenate(src)
    ntile = -(-len(bi) // 32)
    for t in split(bi, x, ntile):
        tx = x[t]
        rel = x[src] - tx[0]
        rel -= np.round(rel)
        sx = tx[0] + rel
        tt = tx
        r2 = ((tt[:, None, :] - sx[None, :, :]) ** 2).sum(-1)
        tot["useful"] += int((r2 < rc * rc).sum())
        def passing(grp):
            lo, hi = tt[grp].min(0), tt[grp].max(0)
            gap = np.maximum(np.maximum(lo - sx, sx - hi), 0)
            return (gap ** 2).sum(1) <= rc * rc
        def staged(grp):
            return int(passing(grp).sum())
        tot["exact"] += 32 * int((r2 < rc * rc).any(0).sum())
        allg = np.arange(len(t))
        tot["tile"] += 32 * staged(allg)
        for G in (2, 4, 8):
            groups = kd_order(allg, tt, {2: 1, 4: 2, 8: 3}[G])
            cnt = [staged(g) for g in groups]
            tot[f"g{G}"] += 32 * max(cnt)
            if G == 4:
                tot["g4s"] += 8 * sum(cnt)   # if groups ran independently
            if G in (4, 8):   # one list, admitted if any group box is in reach
                tot[f"u{G}"] += 32 * int(np.any([passing(g) for g in groups], axis=0).sum())
print({k: round(tot["useful"] / v, 3) for k, v in tot.items() if k != "useful"})
