timeout 120 python -m pytest -q -x -m gpu "tests/test_parity_engine.py::test_smooth_windows" -p no:cacheprovider 2>&1 | tail -2
