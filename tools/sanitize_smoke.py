"""Small end-to-end pass over every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck): compress, negate, scalar add/mul,
element-wise add, hadamard, pair stats, block means, mean, variance,
decompress, .hsz assembly -- on a 3-tile field with a tail block."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2408_11971_b200 as H  # noqa: E402
from paper_2408_11971_b200 import distsim, hszio  # noqa: E402

n = 32 * 128 * int(os.environ.get("HSZ_SAN_TILES", "3")) + 21
i = np.arange(n)
xa = (np.sin(i / 50.0) * 30 + np.random.default_rng(0).normal(0, 0.1, n)).astype(np.float32)
xb = (np.cos(i / 70.0) * 10).astype(np.float32)
ra = H.RawArray(torch.from_numpy(xa).cuda(), (n,), "f32")
rb = H.RawArray(torch.from_numpy(xb).cuda(), (n,), "f32")
p = H.QuantParams(H.resolve_eps(ra, 1e-3, "rel"), (n,), 32, "f32")
a, b = H.compress(ra, p), H.compress(rb, p)
z = H.scalar_mul(H.scalar_add(H.negate(a), 3.5), -1.25)
e = H.elementwise_add(a, b)
h = H.hadamard(a, b)
agg = distsim.aggregate_homomorphic([a, b, z])
print(H.mean(z), H.variance(e), H.covariance(a, b), H.ssim_global(a, b))
print(float(H.block_means(h).sum()), H.decompress(agg).values.sum().item())
print(len(hszio.serialize_device(e)), H.serialize(z.to_host())[:8].hex())
torch.cuda.synchronize()
print("sanitize smoke ok")
