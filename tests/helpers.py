"""Shared test helpers: synthetic windows and error metrics."""
import numpy as np

from oracle import oracle as O


def rel_inf(a, b):
    """||a - b||_inf / ||b||_inf — the reference's gradient convention
    (fdcheck.hpp:184, test_warp.cpp:374-377)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    den = np.abs(b).max() if b.size else 0.0
    if den == 0.0:
        return float(np.abs(a).max()) if a.size else 0.0
    return float(np.abs(a - b).max() / den)


def smooth_window(W, H, B, n, seed=1, window_us=100000, amp=5.0):
    """bench_window semantics (bench.hpp:112-141) plus smooth spatial flow
    variation so that flow Jacobians are nonzero; all values fp32-representable."""
    rng = np.random.default_rng(seed)
    t = np.sort(rng.integers(0, window_us, n)).astype(np.uint64)
    ev = O.make_events(t, rng.integers(0, W, n), rng.integers(0, H, n),
                       np.where(np.arange(n) % 2 == 0, 1, -1))
    edges = O.make_edges(0, window_us, B)
    xs = np.arange(W)[None, :]
    ys = np.arange(H)[:, None]
    uv = np.zeros((B, 2, H, W))
    for b in range(B):
        u0, v0 = rng.uniform(-15, 15, 2)
        uv[b, 0] = u0 + amp * np.sin(0.05 * xs + 0.3 * b) + 0 * ys
        uv[b, 1] = v0 + amp * np.cos(0.04 * ys - 0.2 * b) + 0 * xs
    uv = uv.astype(np.float32).astype(np.float64)
    return O.Window(W, H, edges, ev, uv)


def chain_inputs(W, H, B, n_windows, events_per_window, seed=7, window_us=100000):
    """Chain-level synthetic batch: two-plane depth (1.0 | 3.0) with mild noise,
    per-bin poses, intrinsics (0.9W, 0.9W, (W-1)/2, (H-1)/2); fp32-representable."""
    rng = np.random.default_rng(seed)
    depth = np.empty((n_windows, H, W))
    depth[:, :, : W // 2] = 1.0
    depth[:, :, W // 2:] = 3.0
    depth *= rng.uniform(0.95, 1.05, depth.shape)
    depth = depth.astype(np.float32).astype(np.float64)
    poses = np.empty((n_windows, B, 6))
    poses[..., :3] = np.array([0.001, -0.002, 0.003]) * rng.uniform(0.5, 1.5, (n_windows, B, 3))
    poses[..., 3:] = np.array([0.002, 0.001, 0.0005]) * rng.uniform(0.5, 1.5, (n_windows, B, 3))
    poses = poses.astype(np.float32).astype(np.float64)
    K = np.array([0.9 * W, 0.9 * W, (W - 1) / 2, (H - 1) / 2])
    evs, offs = [], [0]
    for w in range(n_windows):
        n = events_per_window
        t = np.sort(rng.integers(0, window_us, n)).astype(np.uint64)
        evs.append(O.make_events(t, rng.integers(0, W, n), rng.integers(0, H, n),
                                 np.where(np.arange(n) % 2 == 0, 1, -1)))
        offs.append(offs[-1] + n)
    return depth, poses, K, np.concatenate(evs).astype(O.EVENT_DTYPE), np.array(offs, np.uint64)


def contraction_window(W, H, B, n, factor=0.2, seed=11, window_us=100000):
    """Still first half, then a radial flow that shrinks the sensor toward its
    centre by `factor` over the second half: events keep their spread at the
    middle reference (the sort key), and at the last references one 32x16 owner
    tile gathers ~(1/factor)^2 x 8 sort tiles, more than a precomputed list
    holds (kListCapO = 128), so the owner kernels take their overflow
    (box-scan) path."""
    rng = np.random.default_rng(seed)
    t = np.sort(rng.integers(0, window_us, n)).astype(np.uint64)
    ev = O.make_events(t, rng.integers(0, W, n), rng.integers(0, H, n),
                       np.where(np.arange(n) % 2 == 0, 1, -1))
    edges = O.make_edges(0, window_us, B)
    nb = B - B // 2  # the trajectory compounds one linear step per bin
    k = -(1.0 - factor ** (1.0 / nb)) / (window_us * 1e-6 / B)  # 1/s
    xs = np.arange(W)[None, :] - (W - 1) / 2
    ys = np.arange(H)[:, None] - (H - 1) / 2
    uv = np.zeros((B, 2, H, W))
    for b in range(B // 2, B):
        uv[b, 0] = k * xs + 0 * ys
        uv[b, 1] = k * ys + 0 * xs
    uv = uv.astype(np.float32).astype(np.float64)
    return O.Window(W, H, edges, ev, uv)
