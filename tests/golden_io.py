"""Loads the golden fixtures (tests/golden/*.npz, written by make_golden.py)."""
import os

import numpy as np

from oracle import oracle as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
WINDOW_FIXTURES = ["fd_100", "fd_7", "fd_503", "fd_1300", "fd_masked_900", "smooth_32x24"]
CHAIN_FIXTURES = ["chain_1", "chain_20"]


def load(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))


def events_of(d):
    return np.ascontiguousarray(d["events"]).view(O.EVENT_DTYPE).reshape(-1)


def window_of(d):
    return O.Window(int(d["W"]), int(d["H"]), d["edges"], events_of(d), d["flows"])
