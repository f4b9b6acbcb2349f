import numpy as np


def fromhex(xs):
    return np.array([float.fromhex(x) for x in xs], dtype=np.float64)


def profiles_fromhex(ps):
    return [(float.fromhex(p[0]), float.fromhex(p[1]), int(p[2]), int(p[3])) for p in ps]


def bits_equal(a, b):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    return a.shape == b.shape and a.tobytes() == b.tobytes()
