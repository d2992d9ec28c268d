"""CPU: host-side logic of the operator mirror (no device calls)."""
import numpy as np
import pytest

import paper_2412_06359_b200 as P
from oracle import oracle as O


@pytest.mark.parametrize("t0,t1,B", [(0, 100000, 10), (5, 1000007, 7), (0, 3, 3), (123, 124, 1),
                                     (0, 1000000, 32), (17, 100017, 3)])
def test_make_edges_matches_reference_rule(t0, t1, B):
    """FlowSequence::zeros edge rule (types.hpp:293-300)."""
    np.testing.assert_array_equal(P.make_edges(t0, t1, B), O.make_edges(t0, t1, B))


def test_make_edges_rejects_bad_windows():
    with pytest.raises(P.ConfigError):
        P.make_edges(10, 10, 2)
    with pytest.raises(P.ConfigError):
        P.make_edges(0, 10, 0)


def test_flow_sequence_helpers():
    f = P.FlowSequence.zeros(6, 4, 0, 1000, 3)
    assert f.n_bins == 3 and f.width == 6 and f.height == 4
    assert f.t_start_us() == 0 and f.t_end_us() == 1000
    z = f.zeros_like()
    assert z.uv.shape == (3, 2, 4, 6) and not z.uv.any()


@pytest.mark.parametrize("field,value,exc", [
    ("x", [1, 9, 2], P.CoordinateRangeError), ("p", [1, 0, 1], P.InvalidPolarityError),
    ("t_us", [5, 3, 7], P.UnsortedEventsError), ("t_us", [5, 6, 1000], P.TimeRangeError)])
def test_validate_window_taxonomy(field, value, exc):
    ev = O.make_events([5, 6, 7], [1, 2, 3], [1, 2, 3], [1, -1, 1])
    ev[field] = value
    sl = P.EventSlice(8, 8, 0, 1000, ev)
    with pytest.raises(exc):
        P.Engine.validate_window(sl, P.FlowSequence.zeros(8, 8, 0, 1000, 2))


def test_validate_window_flow_errors():
    ev = O.make_events([5], [1], [1], [1])
    sl = P.EventSlice(8, 8, 0, 1000, ev)
    with pytest.raises(P.DimensionMismatchError):
        P.Engine.validate_window(sl, P.FlowSequence.zeros(9, 8, 0, 1000, 2))
    with pytest.raises(P.ConfigError):
        P.Engine.validate_window(sl, P.FlowSequence.zeros(8, 8, 0, 999, 2))
    P.Engine.validate_window(sl, P.FlowSequence.zeros(8, 8, 0, 1000, 2))  # valid


def test_event_slice_counts_torch_bytes():
    import torch
    ev = O.make_events([1, 2], [0, 1], [0, 1], [1, -1])
    sl = P.EventSlice(4, 4, 0, 10, torch.from_numpy(ev.view(np.uint8)))
    assert sl.n_events == 2
