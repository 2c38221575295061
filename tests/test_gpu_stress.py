"""Randomised sequences of every operation in one process (tools/stress.py):
workspace / ticket / epoch state carried across many launches of different
kernels, each result checked bit-exactly against the CPU oracle."""

import os
import sys

import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", [11, 12])
def test_random_operation_sequences(seed):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    import stress

    stress.run(iters=80, seed=seed, verbose=False)
