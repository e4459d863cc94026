"""Output-side kernels on grids with several frame blocks and partial bin tiles.

The statistics refresh (fastfca.py:373-387), the fused Wiener images and the back-transform
(fastfca.py:258-273, wiener.py:38-43) tile bins x frame blocks; small test shapes usually fit one
block.  These shapes force several blocks per tile (a ragged last block included), partial 32-bin
tiles and both kernel families (I <= 4 in registers, 4 < I <= 8 with P / Q in shared memory),
against the fp64 oracle: complex128 rel <= 1e-10, complex64 rel <= 1e-4 (test_gpu_fastfca.py).
"""

import numpy as np
import pytest

from conftest import rel
from oracle import fastfca_ref as ffr
from paper_1805_09498_b200 import ObservationTensor, fastfca, wiener
from paper_1805_09498_b200.workloads import mixture

pytestmark = pytest.mark.gpu

# (I, J, F, N): N / 64 >= 2 frame blocks for I <= 4, N / 32 >= 2 for I > 4; F not a multiple of 32
SHAPES = [(3, 3, 40, 300), (4, 4, 33, 203), (2, 3, 70, 130), (8, 6, 40, 200), (5, 2, 35, 97), (7, 1, 9, 70)]


@pytest.mark.parametrize("dt", ["c128", "c64"])
@pytest.mark.parametrize("I,J,F,N", SHAPES)
def test_stats_images_back_transform_on_multi_block_grids(I, J, F, N, dt):
    y, P0, lam0, v0, _ = mixture(4000 + 10 * I + J, I, J, F, N, 4, 0.0)
    ref = ffr.run_fastfca(y, P0, lam0, v0, iterations=2)
    ref_img = ffr.images(ref.P, ref.mu)
    if dt == "c64":
        y, P0, lam0, v0 = (y.astype(np.complex64), P0.astype(np.complex64), lam0.astype(np.float32),
                           v0.astype(np.float32))
    tol = 1e-10 if dt == "c128" else 1e-4
    run = fastfca.run_fastfca(ObservationTensor(y), fastfca.FastFcaParams(P0, lam0, v0), iterations=2)
    assert rel(run.stats.mu, ref.mu) <= tol
    assert rel(run.stats.phi, ref.phi) <= tol
    fused = fastfca.images_from_state(ObservationTensor(y), run.params)
    assert rel(fused, ref_img) <= 10 * tol
    explicit = wiener.mmse_images_fastfca(run.params, run.stats).stft
    assert rel(explicit, ref_img) <= 10 * tol
    assert rel(explicit, fused) <= 10 * tol
    plain = fastfca.back_transform_means(run.params.P, run.stats.mu)  # (J, N, F, I) layout
    assert rel(np.moveaxis(plain, -1, 1), ref_img) <= 10 * tol
    # Wiener partition (test_wiener.py:56-74): the images of all sources add up to the observation
    assert np.abs(fused.sum(axis=0) - y).max() <= (1e-8 if dt == "c128" else 1e-3) * np.abs(y).max()


@pytest.mark.parametrize("N", [130, 200, 300, 448])
def test_complex128_mid_length_bins(N):
    # regression: for 130 <= N <= 448 the complex128 one-bin plan halved a 160..224-thread CTA to
    # 80..112 threads -- a partial last warp under full-mask shuffles -- and the estimates were
    # off by ~10 %; the plan now rounds to whole warps (CPU check: test_abi_symbols.py)
    y, P0, lam0, v0, _ = mixture(7000 + N, 3, 3, 6, N, 4, 0.0)
    ref = ffr.run_fastfca(y, P0, lam0, v0, iterations=3, record_likelihood=True, stats=False)
    for rec in (False, True):
        run = fastfca.run_fastfca(ObservationTensor(y), fastfca.FastFcaParams(P0, lam0, v0), iterations=3,
                                  record_likelihood=rec)
        assert rel(run.params.P, ref.P) <= 1e-10
        assert rel(run.params.Lam, ref.lam) <= 1e-10
        assert rel(run.params.v, ref.v) <= 1e-10
        if rec:
            assert abs(run.loglik_after_p[-1] - ref.loglik_after_p[-1]) <= 1e-10 * abs(ref.loglik_after_p[-1])
