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


def test_encoder_interleaving():
    """Every look-back encoder interleaved in random order on random sizes
    (grids from 1 CTA to the whole GPU), each launched twice with identical
    bytes required, oracle spot checks, watchdog armed
    (tools/stress_encoders.py; the long run is in profiles/)."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    import stress_encoders

    assert stress_encoders.run(iters=300, seed=5, oracle_every=30, verbose=False) == 300 * 16
