"""Diagnostic (GPU): distinct 128 B lines per warp gather of the (x0, y0) corner at
every reference for the sorted event order vs finer within-tile orders.
Line id of a double2 plane element: (y0 * W + x0) * 16 // 128."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import bench
import paper_2412_06359_b200 as P
from oracle import oracle as O

wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "C"]
depth, poses, K, ev, offs = bench.make_inputs(wl, 0, 1)
W, H, B, t1 = wl["W"], wl["H"], wl["B"], wl["window_us"]
eng = P.Engine()
gf = eng.depth_pose_to_flows(depth[0], poses[0], K, 0, t1)
fwd = eng.forward(P.EventSlice(W, H, 0, t1, ev), gf.flows)
keys, perm, skeys = fwd.sort_products()
tr = fwd.traj
pos = tr.pos  # [n, B+1, 2]
alive = tr.alive.astype(bool)
x0 = np.clip(np.floor(pos[..., 0]), 0, W - 2).astype(np.int64)
y0 = np.clip(np.floor(pos[..., 1]), 0, H - 2).astype(np.int64)
line = (y0 * W + x0) * 16 // 128  # [n, R]
def stats(order, name, group=32):
    o = order[alive[order]]
    m = len(o) // group * group
    o = o[:m].reshape(-1, group)
    res = []
    for r in range(B + 1):
        L = line[o, r]
        Ls = np.sort(L, axis=1)
        d = 1 + (np.diff(Ls, axis=1) != 0).sum(1)
        # per quarter-warp distinct lines, summed over the 4 quarters
        q = 0
        for k in range(4):
            Q = np.sort(L[:, 8 * k:8 * k + 8], axis=1)
            q += (1 + (np.diff(Q, axis=1) != 0).sum(1)).mean()
        res.append((d.mean(), q))
    a = np.array(res)
    print(f"{name:28s} distinct lines/warp: mid {a[B//2,0]:.1f} mean {a[:,0].mean():.1f} | "
          f"sum of quarter-warp lines: mid {a[B//2,1]:.1f} mean {a[:,1].mean():.1f}")
stats(perm.astype(np.int64), "current (tile, time)")
m = B // 2
ym, xm = y0[:, m], x0[:, m]
tile = skeys.astype(np.int64)
sk = np.zeros(len(keys), np.int64); sk[perm] = tile
rowmaj = np.lexsort((xm[perm], ym[perm], sk[perm]))
stats(perm[rowmaj].astype(np.int64), "(tile, y_mid, x_mid)")
morton = lambda x, y: sum((((x >> b) & 1) << (2 * b)) | (((y >> b) & 1) << (2 * b + 1)) for b in range(3))
mk = morton(xm[perm] & 7, ym[perm] & 7)
mo = np.lexsort((mk, sk[perm]))
stats(perm[mo].astype(np.int64), "(tile, morton8)")
glob = np.lexsort((xm, ym))
stats(glob.astype(np.int64), "global (y_mid, x_mid)")
tslot, sub = fwd.sort_order2(len(perm))
stats(perm[tslot].astype(np.int64), "device order2 (approx mid)")
# how far is the approximate mid pixel from the exact one
o2 = perm[tslot].astype(np.int64)
ex = (ym[o2] & 7) * 8 + (xm[o2] & 7)
print("sub-key == exact mid pixel sub-key:", np.mean(ex == sub), " same row:", np.mean((ym[o2] & 7) == (sub >> 3)))
dx = np.abs(np.diff(xm[o2])); dy = np.abs(np.diff(ym[o2]))
print("median |dx|,|dy| between consecutive (exact mid):", np.median(dx), np.median(dy), "mean", dx.mean(), dy.mean())

# ---- owner-kernel bank classes: max lanes per bank class (8y + x) mod 32 of the
# (x0, y0) corner at every reference, 32 consecutive events of one tile
def bank_stats(order, name):
    o = order[alive[order]]
    til = sk[o]
    res = []
    for r in range(B + 1):
        cls = (8 * y0[o, r] + x0[o, r]) % 32
        mx = []
        for g in range(0, len(o) - 32, 32 * 7):
            if til[g] != til[g + 31]:
                continue
            mx.append(np.bincount(cls[g:g + 32], minlength=32).max())
        res.append(np.mean(mx))
    print(f"{name:28s} mean max bank load per 32 lanes: {np.mean(res):.2f} (mid ref {res[B // 2]:.2f})")

cur = perm.astype(np.int64)
bank_stats(cur, "current (tile, time)")
# (tile, j, rank within (j, class), class) with the device's approximate mid pixel
o2t = perm[tslot].astype(np.int64)            # events in device order2 (tile, sub)
cls_dev = np.zeros(len(keys), np.int64)
cls_dev[o2t] = ((8 * (sub >> 3).astype(np.int64) + (sub & 7)) % 32)
jj = tr.bin.astype(np.int64)
def interleaved(cls):
    # within (tile, j) groups in time order: key = (tile, j, k_c, c)
    o = cur
    t_, j_, c_ = sk[o], jj[o], cls[o]
    grp = (t_ * 16 + j_) * 32 + c_
    # rank within (tile, j, class) in time order
    idx = np.argsort(grp, kind="stable")
    g_sorted = grp[idx]
    start = np.r_[0, np.flatnonzero(np.diff(g_sorted)) + 1]
    rank = np.zeros(len(o), np.int64)
    run = np.arange(len(o)) - np.repeat(start, np.diff(np.r_[start, len(o)]))
    rank[idx] = run
    key = (t_ * 16 + j_) * (1 << 20) + rank * 32 + c_
    return o[np.argsort(key, kind="stable")]
bank_stats(interleaved(cls_dev), "(tile, j, k_c, c) approx mid")
cls_ex = (8 * ym + xm) % 32
bank_stats(interleaved(cls_ex), "(tile, j, k_c, c) exact mid")
def interleaved_tile(cls):
    o = cur
    t_, c_ = sk[o], cls[o]
    grp = t_ * 32 + c_
    idx = np.argsort(grp, kind="stable")
    g_sorted = grp[idx]
    start = np.r_[0, np.flatnonzero(np.diff(g_sorted)) + 1]
    run = np.arange(len(o)) - np.repeat(start, np.diff(np.r_[start, len(o)]))
    rank = np.zeros(len(o), np.int64)
    rank[idx] = run
    key = t_ * (1 << 24) + rank * 32 + c_
    return o[np.argsort(key, kind="stable")]
ti = interleaved_tile(cls_dev)
bank_stats(ti, "(tile, k_c, c) approx mid")
stats(ti, "(tile, k_c, c) lines")
