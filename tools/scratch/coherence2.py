"""Diagnostic (GPU for the forward products, then numpy): L1 lines per quarter warp
of the trajectory's flow gathers (plane of bin i at the position the step samples,
as k_traj_records / k_bwd_event walk them: lane-dependent bin j), and owner bank
loads, for several event orders inside sort tiles."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import bench
import paper_2412_06359_b200 as P

wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "C"]
depth, poses, K, ev, offs = bench.make_inputs(wl, 0, 1)
W, H, B, t1 = wl["W"], wl["H"], wl["B"], wl["window_us"]
eng = P.Engine()
gf = eng.depth_pose_to_flows(depth[0], poses[0], K, 0, t1)
fwd = eng.forward(P.EventSlice(W, H, 0, t1, ev), gf.flows)
keys, perm, skeys = fwd.sort_products()
tr = fwd.traj
pos = tr.pos
jj = tr.bin.astype(np.int64)
alive = tr.alive.astype(bool)
x0 = np.clip(np.floor(pos[..., 0]), 0, W - 2).astype(np.int64)
y0 = np.clip(np.floor(pos[..., 1]), 0, H - 2).astype(np.int64)
HW = W * H
sk = np.zeros(len(keys), np.int64)
sk[perm] = skeys
m = B // 2
xm, ym = x0[:, m], y0[:, m]


def lines_traj(order):
    o = order[alive[order]]
    n = len(o) // 32 * 32
    o = o[:n].reshape(-1, 32)
    tot = 0.0
    for s in range(B - 1):
        j = jj[o]
        back = s < j
        i = np.where(back, j - 1 - s, s + 1)
        r = np.where(back, i + 1, i)
        xx = np.take_along_axis(x0[o], r, 1) if False else x0[o, r] if False else None
        px = x0[o[:, :, None], r[:, :, None]][..., 0] if False else x0[o, r]
        py = y0[o, r]
        line = (i * HW + py * W + px) * 16 // 128
        for q in range(4):
            L = np.sort(line[:, 8 * q:8 * q + 8], 1)
            tot += (1 + (np.diff(L, 1) != 0).sum(1)).mean()
    return tot / (B - 1)


def banks(order):
    o = order[alive[order]]
    res = []
    for r in range(B + 1):
        cls = (8 * y0[o, r] + x0[o, r]) % 32
        mx = []
        for g in range(0, len(o) - 32, 32 * 5):
            mx.append(np.bincount(cls[g:g + 32], minlength=32).max())
        res.append(np.mean(mx))
    return np.mean(res)


cur = perm.astype(np.int64)
orders = {
    "(tile, time)": cur,
    "(tile, y_mid, x_mid)": cur[np.lexsort((xm[cur], ym[cur], sk[cur]))],
    "(tile, j, y_mid, x_mid)": cur[np.lexsort((xm[cur], ym[cur], jj[cur], sk[cur]))],
    "(tile, j, morton)": cur[np.lexsort((((ym[cur] & 7) >> 1) * 4 + ((xm[cur] & 7) >> 1), jj[cur], sk[cur]))],
}
for k, o in orders.items():
    print(f"{k:26s} traj quarter-warp lines per step-gather {lines_traj(o):6.2f}   owner max bank load {banks(o):.2f}")
