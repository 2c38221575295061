"""The encoders' look-back watchdog (HSZ_ERR_LOOKBACK_TIMEOUT): a placement
wait that can never be satisfied raises DeviceTimeout on the host instead of
hanging the GPU, and the next operation on the same context is correct again
(the workspace is re-initialised when the error is raised).

The unsatisfiable wait is provoked the way an aborted launch would leave it:
the workspace's tile-ticket counter is bumped before a launch, so tickets
start at 3 -- tiles 0..2 are never encoded and tile 3's look-back waits for
tile 2 forever.  The watchdog bound is lowered for the test
(hsz_set_lookback_watchdog) so it fires within milliseconds."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def H():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2408_11971_b200 as mod

    return mod


def _field(n, seed=0):
    rng = np.random.default_rng(seed)
    return (np.cumsum(rng.normal(0, 0.5, n)) + 100).astype(np.float32)


def _bump_ticket(ctx, v=3):
    import torch

    ctx.stream.synchronize()
    ctx.ws[:8].view(torch.int64)[0] = v
    ctx.stream.synchronize()


@pytest.mark.parametrize("op", ["compress", "scalar_mul", "elementwise_add", "encode_from_quant"])
def test_lookback_timeout_raises_and_recovers(H, op):
    import torch

    from paper_2408_11971_b200 import _native
    from paper_2408_11971_b200.device import context
    from paper_2408_11971_b200.errors import DeviceTimeout

    n = 32 * 128 * 40 + 17                      # 41 tiles
    x = torch.from_numpy(_field(n)).cuda()
    raw = H.RawArray(x, (n,), "f32")
    p = H.QuantParams(1e-3, (n,), 32, "f32")
    s = H.compress(raw, p)
    q = H.decode_to_quant(s)

    def run():
        if op == "compress":
            return H.compress(raw, p)
        if op == "scalar_mul":
            return H.scalar_mul(s, -1.25)
        if op == "elementwise_add":
            return H.elementwise_add(s, s)
        return H.encode_from_quant(q)

    want = H.serialize(run().to_host())
    ctx = context()
    lib = _native.load()
    old = lib.hsz_set_lookback_watchdog(1 << 10)
    try:
        _bump_ticket(ctx)
        with pytest.raises(DeviceTimeout):
            run().check()
    finally:
        lib.hsz_set_lookback_watchdog(old)
    assert lib.hsz_set_lookback_watchdog(0) == old
    # the context recovered: same bytes as before the fault
    assert H.serialize(run().to_host()) == want
    assert ctx.read_flags() == 0
