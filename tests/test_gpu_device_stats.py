"""The device-resident statistics snapshot of run_fastfca (fastfca.py:466 computed in HBM, copied
to the host only when read) and run_fastfca_batch(stats="device"): the same values as the host
path, bitwise, in every copy path (single call, mixture-chunked and F-block-chunked pipelines),
the dataclass contract of TransformedStats, and the Wiener images consuming the snapshot in place."""

import dataclasses
import pickle

import numpy as np
import pytest
import torch

from paper_1805_09498_b200 import ObservationTensor, fastfca, wiener
from paper_1805_09498_b200.workloads import mixture

pytestmark = pytest.mark.gpu


def cast(dt, *arrs):
    if dt == "c128":
        return arrs
    return [a.astype(np.complex64) if np.iscomplexobj(a) else a.astype(np.float32) for a in arrs]


@pytest.mark.parametrize("dt", ["c128", "c64"])
def test_run_fastfca_snapshot_on_device_then_host(dt):
    y, P0, lam0, v0, _ = mixture(31, 3, 3, 40, 90)
    y, P0, lam0, v0 = cast(dt, y, P0, lam0, v0)
    run = fastfca.run_fastfca(ObservationTensor(y), fastfca.FastFcaParams(P0, lam0, v0), iterations=6)
    assert run.stats.device_tensor("mu") is not None and run.stats.device_tensor("phi") is not None
    P, lam, v, _, mu, phi = fastfca.run_fastfca_batch(y[None], P0[None], lam0[None], v0[None], iterations=6,
                                                      stats=True)
    run.params.P[...] = 0  # the snapshot does not follow later changes of the parameters
    assert isinstance(run.stats.mu, np.ndarray) and run.stats.device_tensor("mu") is None
    assert np.array_equal(run.stats.mu, mu[0]) and np.array_equal(run.stats.phi, phi[0])
    assert run.stats.mu.dtype == y.dtype and run.stats.phi.dtype == v0.dtype


def test_snapshot_dataclass_contract():
    y, P0, lam0, v0, _ = mixture(32, 2, 3, 17, 33)
    run = fastfca.run_fastfca(ObservationTensor(y), fastfca.FastFcaParams(P0, lam0, v0), iterations=3)
    d = dataclasses.asdict(run.stats)
    assert isinstance(d["mu"], np.ndarray) and d["mu"].shape == (3, 33, 17, 2)
    run2 = fastfca.run_fastfca(ObservationTensor(y), fastfca.FastFcaParams(P0, lam0, v0), iterations=3)
    rep = dataclasses.replace(run2.stats)  # replace() reads the fields: plain arrays in the copy
    assert isinstance(rep.mu, np.ndarray) and np.array_equal(rep.phi, run2.stats.phi)
    back = pickle.loads(pickle.dumps(run.stats))
    assert np.array_equal(back.mu, run.stats.mu) and np.array_equal(back.phi, run.stats.phi)


@pytest.mark.parametrize("dt", ["c128", "c64"])
def test_images_from_device_snapshot_match_host_stats(dt):
    y, P0, lam0, v0, _ = mixture(33, 3, 3, 40, 90)
    y, P0, lam0, v0 = cast(dt, y, P0, lam0, v0)
    run = fastfca.run_fastfca(ObservationTensor(y), fastfca.FastFcaParams(P0, lam0, v0), iterations=5)
    img_dev = wiener.mmse_images_fastfca(run.params, run.stats).stft  # consumes the device snapshot
    assert run.stats.device_tensor("mu") is not None                   # ... without copying it out
    host = fastfca.TransformedStats(mu=np.array(run.stats.mu), phi=np.array(run.stats.phi))
    img_host = wiener.mmse_images_fastfca(run.params, host).stft
    assert np.array_equal(img_dev, img_host)


@pytest.mark.parametrize("chunks", ["none", "mixtures", "fblocks"])
@pytest.mark.parametrize("dt", ["c128", "c64"])
def test_batch_device_stats_bitwise_host_stats(dt, chunks, monkeypatch):
    U = 1 if chunks == "fblocks" else 3
    ys, Ps, ls, vs = [], [], [], []
    for u in range(U):
        y, P0, lam0, v0, _ = mixture(40 + u, 3, 3, 37, 64)
        ys.append(y), Ps.append(P0), ls.append(lam0), vs.append(v0)
    y, P0, lam0, v0 = cast(dt, np.stack(ys), np.stack(Ps), np.stack(ls), np.stack(vs))
    if chunks == "none":
        monkeypatch.setenv("FFCA_NO_PIPELINE", "1")
    else:  # force the chunked host pipeline at this small size
        monkeypatch.setenv("FFCA_PIPELINE_MIN_BYTES", "1")
        monkeypatch.setenv("FFCA_PIPELINE_CHUNKS", "3")
    Ph, lh, vh, _, muh, phih = fastfca.run_fastfca_batch(y, P0, lam0, v0, iterations=4, stats=True)
    Pd, ld, vd, _, mud, phid = fastfca.run_fastfca_batch(y, P0, lam0, v0, iterations=4, stats="device")
    assert isinstance(mud, torch.Tensor) and mud.is_cuda and phid.is_cuda
    torch.cuda.synchronize()
    assert np.array_equal(Pd, Ph) and np.array_equal(ld, lh) and np.array_equal(vd, vh)
    assert np.array_equal(mud.cpu().numpy(), muh) and np.array_equal(phid.cpu().numpy(), phih)


def test_batch_device_stats_out_validation():
    y, P0, lam0, v0, _ = mixture(50, 3, 3, 9, 20)
    bad = (torch.empty(1), torch.empty(1))
    with pytest.raises(ValueError):
        fastfca.run_fastfca_batch(y[None], P0[None], lam0[None], v0[None], iterations=1, stats="device",
                                  stats_out=bad)


@pytest.mark.parametrize("dt", ["c128", "c64"])
def test_run_fca_statistics_stay_on_device_until_read(dt):
    from paper_1805_09498_b200 import fca
    y, _, _, v0, _ = mixture(34, 3, 3, 21, 50)
    S0 = np.broadcast_to(np.eye(3, dtype=np.complex128), (3, 21, 3, 3)).copy()
    y, S0, v0 = cast(dt, y, S0, v0)
    obs = ObservationTensor(y)
    run = fca.run_fca(obs, fca.FcaParams(S0, v0), iterations=4, record_likelihood=True)
    assert run.stats.device_tensor("mu") is not None and run.stats.device_tensor("phi") is not None
    # the statistics are the E-step at the penultimate parameters (fca.py:211)
    prev = fca.run_fca(obs, fca.FcaParams(S0, v0), iterations=3)
    ref = fca.e_step(prev.params, obs)
    assert np.array_equal(run.stats.mu, ref.mu) and np.array_equal(run.stats.phi, ref.phi)
    assert run.stats.device_tensor("mu") is None and len(run.loglik) == 5
