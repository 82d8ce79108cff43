"""Shared helpers for the test suite."""
import numpy as np


def arr(x, shape=None):
    """Golden-matrix literal -> uint8 array.  `[rows, cols, data]` triples
    carry explicit (possibly zero) shapes."""
    if isinstance(x, list) and len(x) == 3 and isinstance(x[0], int) and isinstance(x[1], int) \
            and isinstance(x[2], list):
        r, c, d = x
        return np.array(d, np.uint8).reshape(r, c)
    a = np.array(x, np.uint8)
    if shape is not None:
        a = a.reshape(shape)
    return a
