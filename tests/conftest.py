"""Shared test plumbing.

* registers the ``gpu`` marker (tests that need a B200 and the built CUDA
  library);
* puts the repo root and ``oracle/`` on ``sys.path`` -- the oracle is test
  infrastructure and is imported only from here, ``smoke()`` and ``bench.py``;
* loads the golden fixtures produced by running the reference itself
  (``tests/golden/make_golden.py``).
"""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden_streams.npz")

#: the FORMAT.md worked example (pkg/FORMAT.md:58-85, tests/conftest.py:8-10)
EXAMPLE_EPS = 0.01
EXAMPLE_VALUES = [-0.025, -0.025, -0.051, -0.052]
EXAMPLE_BINS = [-1, -1, -3, -3]
EXAMPLE_HEX = ("48535a50" "01" "00" "0200" "7b14ae47e17a843f" "20000000"
               "0200000000000000" "0200000000000000" "02" "ffffffff" "20" "08")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 and the built libhsz_b200.so")


class GoldenCase:
    def __init__(self, z, i):
        self.i = i
        self._z = z
        self._p = f"c{i}_"

    def has(self, key):
        return self._p + key in self._z

    def __getitem__(self, key):
        return self._z[self._p + key]

    def s(self, key):
        return str(self[key][0])

    @property
    def eps(self):
        return float(self["eps"][0])

    @property
    def dims(self):
        return tuple(int(d) for d in self["dims"])

    @property
    def block_len(self):
        return int(self["block_len"][0])

    @property
    def dtype(self):
        return "f32" if int(self["dtype"][0]) == 0 else "f64"

    @property
    def kind(self):
        return self.s("kind")

    def raw_values(self):
        v = self["src"]
        return v.astype(np.float32) if self.dtype == "f32" else v.astype(np.float64)

    def bytes_of(self, key):
        return self[key].tobytes()

    def __repr__(self):
        return f"golden#{self.i}({self.kind},{self.dims},k={self.block_len},{self.dtype},eps={self.eps})"


def load_golden():
    z = np.load(GOLDEN)
    return [GoldenCase(z, i) for i in range(int(z["count"][0]))]


@pytest.fixture(scope="session")
def golden_cases():
    return load_golden()
