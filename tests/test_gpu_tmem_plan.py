"""The tensor-memory launch plan of the plain complex64 I = J = 3 loop (run_fastfca, fastfca.py:401-474).

The plan keeps the y records of a CTA's four bins in tensor memory (thread-private columns) and
only the powers in shared memory.  Its arithmetic is that of the 4-bin / 128-thread shared-memory
plan, so the two must agree bit for bit; against the fp64 oracle the complex64 tolerances of
test_gpu_fastfca.py apply (state rel <= 1e-4).
"""

import os

import numpy as np
import pytest

from conftest import rel
from oracle import fastfca_ref as ffr
from paper_1805_09498_b200 import _lib, fastfca
from paper_1805_09498_b200.workloads import mixture

pytestmark = pytest.mark.gpu

ENV = ("FFCA_FORCE_PLAN", "FFCA_NO_TMEM", "FFCA_TMEM_MIN_BINS")


@pytest.fixture(autouse=True)
def _plan_env():
    old = {k: os.environ.pop(k, None) for k in ENV}
    os.environ["FFCA_TMEM_MIN_BINS"] = "0"  # the plan is chosen from one wave of bins on; small cases force it
    yield
    for k in ENV:
        os.environ.pop(k, None)
        if old[k] is not None:
            os.environ[k] = old[k]


def batch(U, F, N, seed, zero_frac=0.0):
    cols = [[], [], [], []]
    for u in range(U):
        y, P0, lam0, v0, _ = mixture(seed + u, 3, 3, F, N, 4, zero_frac)
        for c, a in zip(cols, (y.astype(np.complex64), P0.astype(np.complex64), lam0.astype(np.float32),
                               v0.astype(np.float32))):
            c.append(a)
    return tuple(np.stack(c) for c in cols)


def plan8(U, F, N, lean=1):
    out = np.zeros(8, np.int32)
    assert _lib.load().ffca_plan_loop_ex(0, _lib.C64, U, 3, 3, N, F, _lib.VF_AUTO, lean,
                                         out.ctypes.data_as(_lib._ip)) == 0
    return [int(x) for x in out]


# (U, F, N): single frames, odd frame counts (half-filled last pair), partial 4-bin groups, groups
# straddling mixtures, the 640-frame maximum, more CTAs than fit the device at once
SHAPES = [(1, 5, 24), (2, 7, 1), (1, 9, 2), (1, 3, 3), (3, 11, 151), (1, 4, 640), (2, 6, 639), (1, 513, 626),
          (5, 513, 626)]


@pytest.mark.parametrize("U,F,N", SHAPES)
def test_tmem_plan_bitwise_the_shared_memory_plan(U, F, N):
    p = plan8(U, F, N)
    assert p[0] == 4 and p[3] == 128 and p[6] == 1 and p[7] == 128
    args = batch(U, F, N, 300 + U + F + N)
    run = fastfca.run_fastfca_batch(*args, iterations=6)
    again = fastfca.run_fastfca_batch(*args, iterations=6)
    os.environ["FFCA_FORCE_PLAN"] = "4,1,1,128"  # same CTA shape, y records in shared memory
    smem = fastfca.run_fastfca_batch(*args, iterations=6)
    for a, b, c in zip(run[:3], smem[:3], again[:3]):
        assert np.isfinite(a).all()
        assert np.array_equal(a, b)
        assert np.array_equal(a, c)  # repeated runs: no race on the tensor-memory records


@pytest.mark.parametrize("U,F,N", [(1, 5, 24), (1, 9, 7), (3, 11, 151), (1, 4, 640), (1, 37, 626)])
def test_tmem_plan_against_oracle(U, F, N):
    assert plan8(U, F, N)[6] == 1
    y, P0, lam0, v0 = batch(U, F, N, 900 + N)
    P, lam, v = fastfca.run_fastfca_batch(y, P0, lam0, v0, iterations=8)[:3]
    for u in range(U):
        ref = ffr.run_fastfca(y[u].astype(np.complex128), P0[u].astype(np.complex128), lam0[u].astype(np.float64),
                              v0[u].astype(np.float64), iterations=8, stats=False)
        assert rel(P[u], ref.P) <= 1e-4
        assert rel(lam[u], ref.lam) <= 1e-4
        assert rel(v[u], ref.v) <= 1e-4


def test_tmem_plan_zero_cells_stay_finite():
    # 10 % exactly-zero observation cells (the config-4 edge case of test_gpu_fastfca.py) through
    # the tensor-memory records
    y, P0, lam0, v0 = batch(2, 10, 200, 41, zero_frac=0.1)
    P, lam, v = fastfca.run_fastfca_batch(y, P0, lam0, v0, iterations=10)[:3]
    assert np.isfinite(P).all() and np.isfinite(lam).all() and np.isfinite(v).all() and (v > 0).all()
    ref = ffr.run_fastfca(y[1].astype(np.complex128), P0[1].astype(np.complex128), lam0[1].astype(np.float64),
                          v0[1].astype(np.float64), iterations=10, stats=False)
    assert rel(P[1], ref.P) <= 1e-4 and rel(v[1], ref.v) <= 1e-4


def test_small_batches_keep_the_shared_memory_plan():
    # below one wave of 16 bins per SM the 2-bin shared-memory plan is faster (abi_fastfca.cu plan_loop)
    os.environ.pop("FFCA_TMEM_MIN_BINS")
    assert plan8(1, 513, 626)[6] == 0 and plan8(1, 513, 626)[0] == 2
    assert plan8(256, 513, 626)[6] == 1
    os.environ["FFCA_TMEM_MIN_BINS"] = "0"
    assert plan8(1, 513, 626)[6] == 1


def test_plans_that_do_not_use_tensor_memory():
    # bins longer than 640 frames and the opt-out switch keep the shared-memory plans, which agree with
    # the tensor-memory plan to fp32 regrouping error; the loop with the likelihood record runs the
    # tensor-memory plan too and leaves the estimates of the plain loop unchanged
    assert plan8(1, 6, 642)[6] == 0
    assert plan8(1, 6, 200, lean=0)[6] == 1
    args = batch(2, 6, 200, 17)
    tm = fastfca.run_fastfca_batch(*args, iterations=5)
    full = fastfca.run_fastfca_batch(*args, iterations=5, record_likelihood=True)
    os.environ["FFCA_NO_TMEM"] = "1"
    assert plan8(2, 6, 200)[6] == 0 and plan8(2, 6, 200, lean=0)[6] == 0
    off = fastfca.run_fastfca_batch(*args, iterations=5)
    for a, b, c in zip(tm[:3], full[:3], off[:3]):
        assert rel(a, b) <= 1e-6 and rel(a, c) <= 1e-5
    long_args = batch(1, 6, 642, 23)
    P = fastfca.run_fastfca_batch(*long_args, iterations=3)[0]
    assert np.isfinite(P).all()


# ---------------------------------------------------------------------------
# I = J = 4: cluster plans with the y records in tensor memory (config 2's plan)
# ---------------------------------------------------------------------------


def plan8_44(F, N, lean=1):
    out = np.zeros(8, np.int32)
    assert _lib.load().ffca_plan_loop_ex(0, _lib.C64, 1, 4, 4, N, F, _lib.VF_AUTO, lean,
                                         out.ctypes.data_as(_lib._ip)) == 0
    return [int(x) for x in out]


@pytest.mark.parametrize("N,C", [(2200, 2), (2201, 2), (4101, 2), (8200, 4)])
def test_cluster_tmem_plan_i4(N, C):
    # bins too long for one CTA's shared memory: a C-CTA cluster, 256 tensor-memory columns per CTA;
    # uneven frame splits and odd frame counts (half-filled last pair on one rank)
    F = 3
    p = plan8_44(F, N)
    assert p[0] == 1 and p[1] == C and p[3] == 128 and p[6] == 1 and p[7] == 256
    y, P0, lam0, v0, _ = mixture(500 + N, 4, 4, F, N, 8, 0.0)
    a32 = (y.astype(np.complex64)[None], P0.astype(np.complex64)[None], lam0.astype(np.float32)[None],
           v0.astype(np.float32)[None])
    tm = fastfca.run_fastfca_batch(*a32, iterations=4)[:3]
    again = fastfca.run_fastfca_batch(*a32, iterations=4)[:3]
    os.environ["FFCA_NO_TMEM"] = "1"
    assert plan8_44(F, N)[6] == 0
    sm = fastfca.run_fastfca_batch(*a32, iterations=4)[:3]
    ref = ffr.run_fastfca(y, P0, lam0, v0, iterations=4, stats=False)
    for a, b, c, want in zip(tm, sm, again, (ref.P, ref.lam, ref.v)):
        assert np.array_equal(a, c)
        assert rel(a, b) <= 1e-5
        assert rel(a[0], want) <= 1e-4


@pytest.mark.parametrize("F,N,K", [(6, 151, 1), (5, 640, 1), (7, 33, 2), (4, 2, 1)])
def test_tmem_plan_full_loop_likelihood(F, N, K):
    # the loop with the likelihood record (and inner iterations) on the tensor-memory plan: state and
    # every recorded likelihood against the oracle, and against the shared-memory plan
    assert plan8(1, F, N, lean=0)[6] == 1
    y, P0, lam0, v0, _ = mixture(77 + N, 3, 3, F, N, 4, 0.0)
    a32 = (y.astype(np.complex64)[None], P0.astype(np.complex64)[None], lam0.astype(np.float32)[None],
           v0.astype(np.float32)[None])
    T = 4
    P, lam, v, ll = fastfca.run_fastfca_batch(*a32, iterations=T, inner_iterations=K, record_likelihood=True)
    os.environ["FFCA_NO_TMEM"] = "1"
    Ps, lams, vs, lls = fastfca.run_fastfca_batch(*a32, iterations=T, inner_iterations=K, record_likelihood=True)
    assert rel(P, Ps) <= 1e-5 and rel(v, vs) <= 1e-5
    assert np.max(np.abs(ll - lls) / np.abs(lls)) <= 1e-6
    if N > 3:  # (fewer frames than channels: singular B_i, not an oracle case)
        ref = ffr.run_fastfca(y, P0, lam0, v0, iterations=T, inner_iterations=K, record_likelihood=True, stats=False)
        assert rel(P[0], ref.P) <= 1e-4 and rel(lam[0], ref.lam) <= 1e-4 and rel(v[0], ref.v) <= 1e-4
        want = np.array([ref.loglik_init] + list(ref.loglik_after_em) + list(ref.loglik_after_p))
        got = np.array([ll[0, 0]] + list(ll[0, 1:2 * T + 1:2]) + list(ll[0, 2:2 * T + 1:2]))
        assert np.max(np.abs(got - want) / np.abs(want)) <= 1e-4
