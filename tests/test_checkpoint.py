"""Predictor checkpoints (predictor.hpp:175-218) and the PFM / CSV codecs they use
(io.hpp:178-236, 323-345): host files, checked byte for byte against files the
compiled reference writes and reads."""
import os

import numpy as np
import pytest

import paper_2412_06359_b200 as P
from oracle import oracle as O

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def _pred(seed=3):
    rng = np.random.default_rng(seed)
    params = rng.normal(size=(3, 4)) * 0.7
    poses = np.concatenate([rng.uniform(-0.05, 0.05, (3, 3)), rng.uniform(-0.3, 0.3, (3, 3))], 1)
    poses[1, 4] = 1e-7
    return P.DirectPredictor(params, poses, 8)


def test_pfm_round_trip(tmp_path):
    img = np.arange(12, dtype=np.float32).reshape(3, 4) / 7
    P.write_pfm(img, tmp_path / "a.pfm")
    data = (tmp_path / "a.pfm").read_bytes()
    assert data.startswith(b"Pf\n4 3\n-1.0\n") and len(data) == len(b"Pf\n4 3\n-1.0\n") + 48
    assert np.array_equal(P.read_pfm(tmp_path / "a.pfm"), img)


def test_pfm_errors(tmp_path):
    p = tmp_path / "x.pfm"
    cases = [(b"PF\n2 2\n-1.0\n" + bytes(16), P.BadMagicError),
             (b"Pf\n2 2\n-1.0\n" + bytes(15), P.TruncatedFileError),
             (b"Pf\n2 2\n-1.0\n" + bytes(17), P.IoError),
             (b"Pf\n2 x\n-1.0\n" + bytes(16), P.IoError),
             (b"Pf\n0 2\n-1.0\n", P.DimensionMismatchError),
             (b"Pf\n2 2\n0.0\n" + bytes(16), P.IoError),
             (b"Pf\n2", P.TruncatedFileError)]
    for data, exc in cases:
        p.write_bytes(data)
        with pytest.raises(exc):
            P.read_pfm(p)
    with pytest.raises(P.DimensionMismatchError):
        P.write_pfm(np.zeros((0, 3)), p)


def test_big_endian_and_scaled_pfm(tmp_path):
    img = np.array([[1.5, -2.0], [3.25, 4.0]], np.float32)
    data = b"Pf\n2 2\n2.0\n" + np.ascontiguousarray(img[::-1]).astype(">f4").tobytes()
    (tmp_path / "b.pfm").write_bytes(data)
    assert np.array_equal(P.read_pfm(tmp_path / "b.pfm"), img * np.float32(2.0))


def test_checkpoint_round_trip(tmp_path):
    pred = _pred()
    P.save_predictor(pred, tmp_path / "p.pfm", tmp_path / "p.csv")
    back = P.load_predictor(tmp_path / "p.pfm", tmp_path / "p.csv")
    assert back.upsample == 8
    assert np.array_equal(back.depth_params, pred.depth_params.astype(np.float32).astype(np.float64))
    assert np.array_equal(back.poses, pred.poses)  # shortest round-trip decimal
    lines = (tmp_path / "p.csv").read_text().splitlines()
    assert lines[0] == "bin,upsample,wx,wy,wz,tx,ty,tz" and lines[2].startswith("1,8,")


def test_checkpoint_errors(tmp_path):
    pred = _pred()
    P.save_predictor(pred, tmp_path / "p.pfm", tmp_path / "p.csv")
    csv = tmp_path / "p.csv"
    good = csv.read_text().splitlines()
    for text in ["bin,upsample\n", good[0] + "\n", "\n".join(good[:2] + ["1,8,0,0,0"]) + "\n",
                 "\n".join(good[:2] + ["1,4,0,0,0,0,0,0"]) + "\n"]:
        csv.write_text(text)
        with pytest.raises(P.ConfigError):
            P.load_predictor(tmp_path / "p.pfm", csv)
    bad = P.DirectPredictor(pred.depth_params, pred.poses.copy(), 8)
    bad.poses[0, 0] = 4.0  # rotation angle beyond pi
    with pytest.raises(P.ConfigError):
        P.save_predictor(bad, tmp_path / "q.pfm", tmp_path / "q.csv")


@needs_ref
def test_checkpoint_files_identical_to_reference(tmp_path):
    for seed in (3, 4, 5):
        pred = _pred(seed)
        O.ref_save_predictor(pred.depth_params, 8, pred.poses, tmp_path / "r.pfm", tmp_path / "r.csv")
        P.save_predictor(pred, tmp_path / "m.pfm", tmp_path / "m.csv")
        assert (tmp_path / "r.pfm").read_bytes() == (tmp_path / "m.pfm").read_bytes()
        assert (tmp_path / "r.csv").read_bytes() == (tmp_path / "m.csv").read_bytes()
        params, f, poses = O.ref_load_predictor(tmp_path / "m.pfm", tmp_path / "m.csv")
        mine = P.load_predictor(tmp_path / "r.pfm", tmp_path / "r.csv")
        assert f == mine.upsample and np.array_equal(params, mine.depth_params)
        assert np.array_equal(poses, mine.poses)
        assert np.array_equal(O.ref_read_pfm(tmp_path / "m.pfm"), P.read_pfm(tmp_path / "r.pfm"))


@needs_ref
def test_pfm_error_classes_match_reference(tmp_path):
    p = tmp_path / "x.pfm"
    codes = {P.BadMagicError: 10, P.TruncatedFileError: 11, P.IoError: 12,
             P.DimensionMismatchError: 2}
    for data in [b"PF\n2 2\n-1.0\n" + bytes(16), b"Pf\n2 2\n-1.0\n" + bytes(15),
                 b"Pf\n2 2\n-1.0\n" + bytes(17), b"Pf\n2 x\n-1.0\n", b"Pf\n0 2\n-1.0\n",
                 b"Pf\n2 2\n0\n" + bytes(16), b"Pf\n2", b"Pf 2 2 -1.0 " + bytes(16),
                 b"Pf\n2 2\n-1.0e0\n" + bytes(16), b"Pf\n2 2\n1.5x\n" + bytes(16)]:
        p.write_bytes(data)
        try:
            O.ref_read_pfm(p)
            ref = 0
        except O.OracleError as e:
            ref = e.code
        try:
            P.read_pfm(p)
            mine = 0
        except P.Error as e:
            mine = next(c for k, c in codes.items() if type(e) is k)
        assert ref == mine, (data, ref, mine)
