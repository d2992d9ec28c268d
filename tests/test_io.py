"""Event ingestion: EVT1 files (io.hpp:106-172) and the
window cut that feeds the batched chain.

Pinning: the oracle's EVT1 restatement is checked against the golden files the
reference wrote (tests/golden/evt1/, make_golden.py) and, where the compiled
reference is present, against the reference itself on fuzzed files. The GPU
tests then check the product (host header parse + device record validation +
device window search) against the golden outcomes and the oracle.
"""
import os

import numpy as np
import pytest

import paper_2412_06359_b200 as P
from oracle import oracle as O
from tests.golden_io import GOLDEN
from tests.helpers import chain_inputs

EVT1_DIR = os.path.join(GOLDEN, "evt1")
FILES = ["empty", "three", "random_2k", "bad_magic", "trunc_record", "trunc_header",
         "unsorted", "coord_at_width", "zero_polarity", "trailing", "zero_width"]
HEADER_ERRORS = {"bad_magic": P.BadMagicError, "trunc_record": P.TruncatedFileError,
                 "trunc_header": P.TruncatedFileError, "trailing": P.IoError,
                 "zero_width": P.DimensionMismatchError}
CLASS_OF = {2: P.DimensionMismatchError, 3: P.CoordinateRangeError, 4: P.InvalidPolarityError,
            5: P.UnsortedEventsError, 6: P.TimeRangeError, 10: P.BadMagicError,
            11: P.TruncatedFileError, 12: P.IoError}
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def _golden():
    return dict(np.load(os.path.join(GOLDEN, "evt1.npz")))


def _path(name):
    return os.path.join(EVT1_DIR, name + ".evt1")


def _events(raw):
    return np.ascontiguousarray(raw).view(O.EVENT_DTYPE).reshape(-1)


# ---------------------------------------------------------------------------
# CPU: oracle pinning and host logic


@pytest.mark.parametrize("name", FILES)
def test_oracle_read_matches_golden(name):
    g = _golden()
    code = int(g[name + "_code"])
    if code:
        with pytest.raises(O.OracleError) as ei:
            O.read_events(_path(name))
        assert ei.value.code == code
        return
    W, H, t0, t1, ev = O.read_events(_path(name))
    assert [W, H, t0, t1] == [int(v) for v in g[name + "_hdr"]]
    assert np.array_equal(ev, _events(g[name + "_events"]))


@pytest.mark.parametrize("name", ["empty", "three", "random_2k"])
def test_oracle_write_reproduces_reference_file(name, tmp_path):
    g = _golden()
    W, H, t0, t1 = [int(v) for v in g[name + "_hdr"]]
    if name == "empty":
        W, H = 32, 24  # written with the header dims of test_core_io.cpp:47-49
    p = tmp_path / "out.evt1"
    O.write_events(p, W, H, t0, t1, _events(g[name + "_events"]))
    assert p.read_bytes() == open(_path(name), "rb").read()


@needs_ref
def test_oracle_read_matches_reference_fuzzed(tmp_path):
    """Random byte patches of reference-written files: same outcome (error code
    or parsed slice) from the restatement and from the reference."""
    rng = np.random.default_rng(5)
    base = [open(_path(n), "rb").read() for n in ("three", "random_2k")]
    p = str(tmp_path / "f.evt1")
    for it in range(300):
        b = bytearray(base[it % 2])
        for _ in range(int(rng.integers(1, 4))):
            k = int(rng.integers(0, len(b)))
            b[k] = int(rng.integers(0, 256))
        if it % 7 == 0:
            b = b[: int(rng.integers(0, len(b) + 1))]
        open(p, "wb").write(bytes(b))
        try:
            ref = ("ok",) + O.ref_read_events(p)
        except O.OracleError as e:
            ref = ("err", e.code)
        try:
            mine = ("ok",) + O.read_events(p)
        except O.OracleError as e:
            mine = ("err", e.code)
        assert ref[0] == mine[0], (ref, mine)
        if ref[0] == "err":
            assert ref[1] == mine[1]
        else:
            assert ref[1:5] == mine[1:5] and np.array_equal(ref[5], mine[5])


@needs_ref
def test_oracle_validate_matches_reference():
    rng = np.random.default_rng(9)
    for it in range(200):
        n = int(rng.integers(0, 40))
        t = np.sort(rng.integers(10, 1000, n)).astype(np.uint64)
        ev = O.make_events(t, rng.integers(0, 12, n), rng.integers(0, 9, n),
                           rng.choice([1, -1, 0, 2], n, p=[0.47, 0.47, 0.03, 0.03]))
        if n > 2 and it % 3 == 0:
            i = int(rng.integers(1, n))
            ev["t_us"][i] = ev["t_us"][i - 1] - 1
        t0, t1 = int(rng.integers(0, 20)), int(rng.integers(900, 1100))
        ref = O.ref_validate_slice(11, 8, t0, t1, ev)
        fv = O.first_violation(ev, 11, 8, (t0, t1))
        assert ref == (fv[1] if fv else 0)


@pytest.mark.parametrize("name", sorted(HEADER_ERRORS))
def test_header_errors_raise_reference_classes(name):
    """Header checks run on the host before any device work (io.hpp:120-134)."""
    with pytest.raises(HEADER_ERRORS[name]):
        P.read_events(_path(name))
    assert issubclass(P.BadMagicError, P.IoError) and issubclass(P.TruncatedFileError, P.IoError)


def test_missing_file_is_io_error(tmp_path):
    with pytest.raises(P.IoError):
        P.read_events(tmp_path / "nope.evt1")


def test_windows_view_host_logic():
    ev = O.make_events(np.arange(0, 1000, 10), np.zeros(100), np.zeros(100), np.ones(100))
    s = P.EventSlice(4, 4, 0, 1000, ev)
    offs = O.window_offsets(ev, 0, 250, 4)
    w = P.Windows(s, 0, 250, offs)
    assert w.n_windows == 4
    for i in range(4):
        sub = w.window(i)
        assert (sub.t_start_us, sub.t_end_us) == (250 * i, 250 * i + 250)
        assert sub.n_events == 25 and np.all(sub.events["t_us"] >= 250 * i)
    with pytest.raises(P.ConfigError):
        w.window(4)


# ---------------------------------------------------------------------------
# GPU: the product


@pytest.mark.gpu
@pytest.mark.parametrize("device", [False, True])
@pytest.mark.parametrize("name", FILES)
def test_read_events_matches_reference(name, device):
    g = _golden()
    code = int(g[name + "_code"])
    if code:
        with pytest.raises(CLASS_OF[code]):
            P.read_events(_path(name), device=device)
        return
    s = P.read_events(_path(name), device=device)
    assert [s.width, s.height, s.t_start_us, s.t_end_us] == [int(v) for v in g[name + "_hdr"]]
    ev = s.events
    if device:
        assert ev.is_cuda
        ev = ev.cpu().numpy().reshape(-1).view(P.EVENT_DTYPE)
    assert np.array_equal(ev, _events(g[name + "_events"]))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["empty", "three", "random_2k"])
@pytest.mark.parametrize("device", [False, True])
def test_write_read_round_trip_is_file_identical(name, device, tmp_path):
    """Evt1.RandomRoundTrip10kEvents (test_core_io.cpp:138-150): read -> write
    reproduces the reference's file byte for byte."""
    s = P.read_events(_path(name), device=device)
    if name == "empty":
        s = P.EventSlice(32, 24, 0, 0)
    p = tmp_path / "rt.evt1"
    P.write_events(s, p)
    assert p.read_bytes() == open(_path(name), "rb").read()


@pytest.mark.gpu
def test_write_events_validates_like_reference(tmp_path):
    """SliceValidate.RejectsInvalidStates (test_core_io.cpp:152-165) through write_events."""
    three = O.make_events([100, 250, 400], [1, 3, 9], [2, 4, 7], [1, -1, 1])
    cases = []
    e = three.copy(); e["p"][1] = 0; cases.append((e, 100, 401, P.InvalidPolarityError))
    e = three[[2, 1, 0]].copy(); cases.append((e, 100, 401, P.UnsortedEventsError))
    cases.append((three.copy(), 100, 400, P.TimeRangeError))
    e = three.copy(); e["x"][0] = 10; cases.append((e, 100, 401, P.CoordinateRangeError))
    cases.append((three.copy(), 401, 100, P.TimeRangeError))
    for ev, t0, t1, cls in cases:
        with pytest.raises(cls):
            P.write_events(P.EventSlice(10, 8, t0, t1, ev), tmp_path / "x.evt1")
        fv = O.first_violation(ev, 10, 8, (t0, t1))
        assert fv is None or CLASS_OF[fv[1]] is cls
    with pytest.raises(P.DimensionMismatchError):
        P.write_events(P.EventSlice(0, 8, 100, 401, three), tmp_path / "x.evt1")


@pytest.mark.gpu
@pytest.mark.parametrize("device", [False, True])
def test_validate_first_violation_at_scale(device):
    """Several violations in a large slice: the device reports the FIRST record
    and, for it, the first failed check (the reference's sequential order)."""
    import torch
    eng = P.Engine()
    rng = np.random.default_rng(3)
    n = 3_000_000
    t = np.sort(rng.integers(0, 10**7, n)).astype(np.uint64)
    base = O.make_events(t, rng.integers(0, 640, n), rng.integers(0, 480, n),
                         np.where(rng.uniform(size=n) < 0.5, 1, -1))
    for trial in range(6):
        ev = base.copy()
        for k in rng.choice(n - 1, 3, replace=False) + 1:
            kind = int(rng.integers(0, 4))
            if kind == 0:
                ev["x"][k] = 640
            elif kind == 1:
                ev["p"][k] = 0
            elif kind == 2:
                ev["t_us"][k] = ev["t_us"][k - 1] - 1 if ev["t_us"][k - 1] else 0
            else:
                ev["y"][k] = 480
                ev["p"][k] = 3  # coordinate wins over polarity on the same record
        fv = O.first_violation(ev, 640, 480, (0, 10**7))
        arr = torch.from_numpy(ev.view(np.uint8).reshape(-1, 16)).cuda() if device else ev
        s = P.EventSlice(640, 480, 0, 10**7, arr)
        if fv is None:
            eng.validate_slice(s)
            continue
        with pytest.raises(CLASS_OF[fv[1]]) as ei:
            eng.validate_slice(s)
        assert f"record {fv[0]} " in str(ei.value)
    eng.validate_slice(P.EventSlice(640, 480, 0, 10**7, base))  # clean slice passes


@pytest.mark.gpu
@pytest.mark.parametrize("device", [False, True])
def test_window_offsets_match_oracle(device):
    import torch
    eng = P.Engine()
    rng = np.random.default_rng(4)
    n = 2_000_000
    t = np.sort(rng.integers(5_000, 3_000_000, n)).astype(np.uint64)
    t[1000:1100] = t[1000]  # runs of equal timestamps at a boundary
    ev = O.make_events(t, np.zeros(n), np.zeros(n), np.ones(n))
    arr = torch.from_numpy(ev.view(np.uint8).reshape(-1, 16)).cuda() if device else ev
    for t0, wl, nw in [(0, 100_000, 31), (int(t[1000]), 7, 1000), (5_000_000, 1000, 3),
                       (int(t[0]), 2_995_000, 1), (0, 1, 1)]:
        got = eng.window_offsets(arr, t0, wl, nw)
        assert np.array_equal(got, O.window_offsets(ev, t0, wl, nw)), (t0, wl, nw)
    empty = np.zeros(0, P.EVENT_DTYPE)
    assert np.array_equal(eng.window_offsets(empty, 0, 10, 3), np.zeros(4, np.uint64))
    with pytest.raises(P.ConfigError):
        eng.window_offsets(ev, 0, 0, 3)


@pytest.mark.gpu
@pytest.mark.parametrize("device", [False, True])
def test_stream_windows_feed_chain(device, tmp_path):
    """EVT1 stream -> read (host or device) -> slice_windows -> chain_batch with a
    per-window clock shift equals (a) chain_batch on the same windows moved onto
    one clock (bit-identical: only the clock differs) and (b) the oracle chain."""
    import torch
    W, H, B, nw, n, wl = 64, 48, 5, 4, 3000, 100_000
    depth, poses, K, ev, offs = chain_inputs(W, H, B, nw, n, seed=12, window_us=wl)
    stream = ev.copy()
    for w in range(nw):  # window w's events move to [w*wl, (w+1)*wl) + 1000
        stream["t_us"][int(offs[w]):int(offs[w + 1])] += np.uint64(1000 + w * wl)
    p = tmp_path / "stream.evt1"
    O.write_events(p, W, H, 1000, 1000 + nw * wl, stream)
    eng = P.Engine(P.EngineOptions(algo="owner"))
    s = P.read_events(p, device=device, engine=eng)
    wins = P.slice_windows(s, wl, t0_us=1000, engine=eng)
    assert wins.n_windows == nw and np.array_equal(wins.offsets, offs)
    dep = torch.from_numpy(depth).cuda() if device else depth
    pos = torch.from_numpy(poses).cuda() if device else poses
    loss, dd, dp = wins.chain_batch(eng, dep, pos, K, out_device=False)
    evs = torch.from_numpy(ev.view(np.uint8).reshape(-1, 16)).cuda() if device else ev
    l1, dd1, dp1 = eng.chain_batch(dep, pos, K, 0, wl, evs, offs, out_device=False)
    assert np.array_equal(loss, l1)
    assert np.array_equal(dd, dd1) and np.array_equal(dp, dp1)
    for w in range(nw):
        fl, _ = O.depth_pose_to_flows(depth[w], poses[w], K, 0, wl)
        win = O.Window(W, H, O.make_edges(0, wl, B), ev[int(offs[w]):int(offs[w + 1])], fl)
        f = O.forward(win)
        assert abs(loss[w] - f["loss"]) <= 1e-5 * abs(f["loss"])
    # a window edge that misses the stream clock is a TimeRangeError, as in the reference
    with pytest.raises(P.TimeRangeError):
        eng.chain_batch(depth, poses, K, 0, wl, stream, offs, window_stride_us=wl)
