"""The reference generator on the device (xmoe_rng_uniform /
xmoe_make_layer_weights) against the compiled reference's Rng
(rng.hpp:24-61) and make_layer_weights (padded_pipeline.cpp:13-27): every
output bit-identical, at any offset (GF(2) jump-ahead across 2^16-output
chains), so the bench's two arms draw identical synthetic inputs."""
import numpy as np
import pytest
import torch

from tests.gpu_util import host

pytestmark = pytest.mark.gpu


def test_rng_known_answer():
    """test_kernels.cpp:98-108: Rng(42).next_u64() == 6667968346354703667;
    uniform() = (x >> 11) * 2^-53."""
    from paper_2508_13337_b200 import capi
    ctx = capi.Context(0, 1, -1)
    u = host(ctx.rng_uniform(42, 0, 1, 0.0, 1.0))[0]
    assert u == (6667968346354703667 >> 11) * 2.0 ** -53


@pytest.mark.parametrize("seed,offset,n", [(0, 0, 1000), (7, 65530, 20), (123, 3 * 65536 + 11, 70000),
                                          (2 ** 63 + 5, 1, 131073)])
def test_rng_stream_vs_reference(ref, seed, offset, n):
    from paper_2508_13337_b200 import capi
    ctx = capi.Context(0, 1, -1)
    want = ref.rng_uniform(seed, offset + n, -1.0, 1.0)[offset:]
    got = host(ctx.rng_uniform(seed, offset, n, -1.0, 1.0))
    assert np.array_equal(got, want)
    # snapped to the bf16-exact token grid, and stored as bf16 / f32
    g = host(ctx.rng_uniform(seed, offset, n, -1.0, 1.0, grid=128.0))
    assert np.array_equal(g, np.round(want * 128) / 128)
    b = ctx.rng_uniform(seed, offset, n, -1.0, 1.0, grid=128.0, dtype=capi.BF16)
    assert np.array_equal(host(b), np.round(want * 128) / 128)
    f = ctx.rng_uniform(seed, offset, n, -1.0, 1.0, dtype=capi.F32)
    assert np.array_equal(host(f), want.astype(np.float32).astype(np.float64))


def test_make_layer_weights_vs_reference(ref):
    from paper_2508_13337_b200 import capi
    ctx = capi.Context(0, 1, -1)
    E, H, F = 8, 24, 40
    seed = ref.salt_seed(0, 7000)
    g, w1, w2 = ref.make_layer_weights(seed, E, H, F)
    dg, d1, d2 = ctx.make_layer_weights(seed, E, H, F)
    assert np.array_equal(host(dg), g) and np.array_equal(host(d1), w1) and np.array_equal(host(d2), w2)
    # an expert slice (one rank's block) and the gate on the 2^-10 grid
    dg, d1, d2 = ctx.make_layer_weights(seed, E, H, F, first_expert=3, n_experts=2, gate_grid=1024.0,
                                        dtype=capi.BF16)
    assert np.array_equal(host(dg), np.round(g * 1024) / 1024)
    assert np.array_equal(host(d1), torch.from_numpy(w1[3:5]).to(torch.bfloat16).double().numpy())
    assert np.array_equal(host(d2), torch.from_numpy(w2[3:5]).to(torch.bfloat16).double().numpy())
