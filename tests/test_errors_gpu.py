"""Error taxonomy through the C-ABI (types.hpp:18-76, engine.hpp:215-222)."""
import numpy as np
import pytest

import paper_2412_06359_b200 as P
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _win(ev, W=8, H=8, t1=1000, B=2):
    return P.EventSlice(W, H, 0, t1, ev), P.FlowSequence(O.make_edges(0, t1, B), np.zeros((B, 2, H, W)))


@pytest.mark.parametrize("mutate,exc", [
    (lambda e: e.__setitem__("x", [1, 9, 2]), P.CoordinateRangeError),
    (lambda e: e.__setitem__("p", [1, 0, 1]), P.InvalidPolarityError),
    (lambda e: e.__setitem__("t_us", [5, 3, 7]), P.UnsortedEventsError),
    (lambda e: e.__setitem__("t_us", [5, 6, 1000]), P.TimeRangeError),
])
def test_event_errors(engine, mutate, exc):
    ev = O.make_events([5, 6, 7], [1, 2, 3], [1, 2, 3], [1, -1, 1])
    mutate(ev)
    sl, fl = _win(ev)
    with pytest.raises(exc):
        engine.forward(sl, fl)
    with pytest.raises(exc):
        P.Engine.validate_window(sl, fl)


def test_first_violation_wins(engine):
    # event 1 has a bad coordinate, event 2 a bad polarity: CoordinateRangeError
    ev = O.make_events([5, 6, 7], [1, 9, 2], [1, 1, 1], [1, 1, 3])
    with pytest.raises(P.CoordinateRangeError):
        engine.forward(*_win(ev))


def test_flow_errors(engine):
    ev = O.make_events([5], [1], [1], [1])
    sl = P.EventSlice(8, 8, 0, 1000, ev)
    with pytest.raises(P.ConfigError):  # edges do not span the slice
        engine.forward(sl, P.FlowSequence(O.make_edges(0, 999, 2), np.zeros((2, 2, 8, 8))))
    with pytest.raises(P.ConfigError):  # non-increasing edges
        engine.forward(sl, P.FlowSequence(np.array([0, 500, 500, 1000], np.uint64),
                                          np.zeros((3, 2, 8, 8))))
    with pytest.raises(P.DimensionMismatchError):
        engine.forward(P.EventSlice(0, 8, 0, 1000, ev), P.FlowSequence(O.make_edges(0, 1000, 2),
                                                                       np.zeros((2, 2, 8, 8))))


def test_rsat_empty(engine):
    with pytest.raises(P.EmptySliceError):
        P.rsat(P.EventSlice(8, 8, 0, 1000), P.FlowSequence(O.make_edges(0, 1000, 1),
                                                             np.zeros((1, 2, 8, 8))))
