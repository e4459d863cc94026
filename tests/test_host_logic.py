"""Host-side logic of the drop-in boundary (CPU only): layouts, dtype policy, argument mapping."""

import numpy as np
import pytest

from paper_1805_09498_b200 import _lib, errors, fastfca, fca
from paper_1805_09498_b200.evalkit import OpCounters, expected_counts
from paper_1805_09498_b200.stft import ObservationTensor
from paper_1805_09498_b200.workloads import CONFIGS, mixture


def test_observation_dtype_policy():
    z = np.ones((2, 3, 4), np.complex64)
    assert ObservationTensor(z).data.dtype == np.complex64  # kept (documented extension)
    assert ObservationTensor(z.astype(np.complex128)).data.dtype == np.complex128
    assert ObservationTensor(np.ones((2, 3, 4))).data.dtype == np.complex128  # coerced as stft.py:63
    with pytest.raises(errors.DimensionMismatch):
        ObservationTensor(np.ones((2, 3)))
    bad = np.ones((2, 3, 4), complex)
    bad[0, 0, 0] = np.nan
    with pytest.raises(ValueError):
        ObservationTensor(bad)


def test_params_validation_matches_reference_errors():
    P = np.broadcast_to(np.eye(3), (5, 3, 3))
    with pytest.raises(errors.DimensionMismatch):
        fastfca.FastFcaParams(P, np.ones((2, 4, 3)), np.ones((2, 6, 5)))
    with pytest.raises(errors.DimensionMismatch):
        fastfca.FastFcaParams(P, np.ones((2, 5, 3)), np.ones((3, 6, 5)))
    with pytest.raises(errors.DimensionMismatch):
        fastfca.FastFcaParams(P, np.ones((2, 5, 3)), np.ones((2, 6, 4)))
    p = fastfca.FastFcaParams(P, np.ones((2, 5, 3)), np.ones((2, 6, 5)))
    assert p.P.dtype == np.complex128 and p.Lam.dtype == np.float64
    assert (p.sources, p.bins, p.order) == (2, 5, 3)
    p32 = fastfca.FastFcaParams(P.astype(np.complex64), np.ones((2, 5, 3)), np.ones((2, 6, 5)))
    assert p32.Lam.dtype == np.float32 and p32.v.dtype == np.float32
    with pytest.raises(errors.DimensionMismatch):
        fca.FcaParams(np.ones((2, 5, 3, 2)), np.ones((2, 6, 5)))


def test_v_floor_argument_mapping():
    J, N, F = 2, 6, 5
    assert fastfca._floor_args(None, J, N, F, False)[0] == _lib.VF_AUTO
    m, s, a = fastfca._floor_args(0.25, J, N, F, False)
    assert m == _lib.VF_SCALAR and s == 0.25 and a is None
    m, _, a = fastfca._floor_args(np.arange(F, dtype=float), J, N, F, True)
    assert m == _lib.VF_BIN and a.dtype == np.float32 and a.shape == (F,)
    m, _, a = fastfca._floor_args(np.ones((J, 1, F)), J, N, F, False)
    assert m == _lib.VF_FULL and a.shape == (J, N, F)


def test_expected_counts_paper_values():
    # PAPER.md:195-199,386-393 at I=J=3, N=249, F=512
    assert expected_counts("fca", 3, 3, 249, 512).inversions == 129024
    assert expected_counts("fca", 3, 3, 249, 512).matmuls == 764928
    assert expected_counts("fastfca", 3, 3, 249, 512, 1).inversions == 2048
    c = OpCounters()
    c.add_inversions(3)
    c.merge(OpCounters(2, 5))
    assert c.as_dict() == {"inversions": 5, "matmuls": 5}
    with pytest.raises(ValueError):
        expected_counts("nope", 1, 1, 1, 1)


def test_generator_shapes_and_determinism():
    y, P0, lam0, v0, vt = mixture(3, 3, 2, 7, 11, 4, 0.1)
    assert y.shape == (3, 11, 7) and P0.shape == (7, 3, 3) and lam0.shape == (2, 7, 3) and v0.shape == (2, 11, 7)
    y2 = mixture(3, 3, 2, 7, 11, 4, 0.1)[0]
    assert np.array_equal(y, y2)
    assert (vt == 0).any()  # sparse-activity cells present
    assert np.allclose(P0, np.eye(3)) and (lam0 == 1).all()
    assert CONFIGS[3].point_iterations == 256 * 626 * 513 * 20


def test_channel_mismatch_raises_before_any_device_call():
    obs = ObservationTensor(np.ones((2, 3, 4), complex))
    params = fastfca.FastFcaParams(np.broadcast_to(np.eye(3), (4, 3, 3)), np.ones((1, 4, 3)), np.ones((1, 3, 4)))
    with pytest.raises(errors.DimensionMismatch):
        fastfca.run_fastfca(obs, params, iterations=1)


# The reference package's public names (fcasep/__init__.py:11-58) and the module-level functions of
# the modules on the path; the drop-in must expose every one of them.
REF_EXPORTS = ["ChannelCountMismatch", "ChannelLengthMismatch", "DimensionMismatch", "EvalReport", "FcaParams",
               "FcasepError", "FastFcaParams", "LengthMismatch", "NotPositiveDefinite", "ObservationTensor",
               "OpCounters", "PosteriorStats", "SampleRateMismatch", "SingularP", "SingularWeightedCovariance",
               "StftConfig", "TooShort", "TransformedStats", "ZeroReference", "analyze", "compute_sdr",
               "expected_counts", "measure_rtf", "run_fca", "run_fastfca", "synthesize"]
REF_MODULE_API = {
    "fastfca": ["FastFcaParams", "TransformedStats", "FastFcaRun", "transform_observations",
                "reconstruct_spatial_covariances", "reconstruct_spatial_covariance", "mixture_weights", "e_step_diag",
                "m_step_diag", "fixed_point_update_P", "log_likelihood", "back_transform_means",
                "back_transform_stats", "params_from_covariances", "run_fastfca"],
    "fca": ["FcaParams", "PosteriorStats", "FcaRun", "power_floor", "mix_covariance", "log_likelihood", "e_step",
            "m_step", "run_fca"],
    "wiener": ["SeparatedImages", "mmse_images_fca", "mmse_images_fastfca", "resynthesize_images"],
    "stft": ["StftConfig", "ObservationTensor", "analyze", "synthesize", "interior_slice"],
    "scene": ["INIT_LOADING", "oracle_covariances", "diffuse_covariances", "init_oracle", "init_diffuse",
              "reference_tensors"],
    "evalkit": ["OpCounters", "expected_counts", "compute_sdr", "rtf_value", "measure_rtf", "EvalReport"],
}


def test_drop_in_exports_every_reference_name():
    import importlib

    import paper_1805_09498_b200 as pkg

    assert [n for n in REF_EXPORTS if not hasattr(pkg, n)] == []
    for mod, names in REF_MODULE_API.items():
        m = importlib.import_module(f"paper_1805_09498_b200.{mod}")
        assert [n for n in names if not hasattr(m, n)] == [], mod


def test_eval_report_rows_and_summary():
    from paper_1805_09498_b200.evalkit import EvalReport, OpCounters

    r = EvalReport("fastfca", 3, 3, 249, 512, 20, 1, 1e-4, [5.0, 7.0], OpCounters(40960, 0), trial=1, seed=3,
                   extras={"rtf_ratio_measured": "1.3"})
    row = r.row()
    assert row["sdr_mean"] == "6.000000" and row["sdr_2"] == "7.000000" and row["inversions"] == 40960
    assert row["rtf_ratio_measured"] == "1.3" and "fastfca: I=3 J=3" in r.summary()


def test_batch_entry_validates_before_the_abi():
    # run_fastfca_batch checks dtypes / shapes / out buffers on the host before any C-ABI call
    y = np.ones((2, 3, 5, 4), np.complex128)
    P0 = np.broadcast_to(np.eye(3), (2, 4, 3, 3)).astype(np.complex64)
    lam0 = np.ones((2, 2, 4, 3), np.float32)
    v0 = np.ones((2, 2, 5, 4), np.float32)
    with pytest.raises(errors.DimensionMismatch):
        fastfca.run_fastfca_batch(np.ones((2, 3, 5, 4)), P0, lam0, v0)  # real y
    with pytest.raises(errors.DimensionMismatch):
        fastfca.run_fastfca_batch(y, P0[:, :3], lam0, v0)
    bad_out = (np.empty((2, 4, 3, 3), np.complex64), np.empty((2, 2, 4, 3)), np.empty((2, 2, 5, 4)))
    with pytest.raises(ValueError):  # complex128 y -> complex128 P out expected
        fastfca.run_fastfca_batch(y, P0, lam0, v0, out=bad_out)
    short = (np.empty((2, 4, 3, 3), np.complex128), np.empty((2, 2, 4, 3)), np.empty((1, 2, 5, 4)))
    with pytest.raises(ValueError):
        fastfca.run_fastfca_batch(y, P0, lam0, v0, out=short)


def test_cli_device_option_parsing():
    from paper_1805_09498_b200 import cli as dev_cli

    class Fake:  # stands in for fcasep.cli: records the argv it is handed and the installed hooks
        _run_estimator = _images_from_run = None

        @staticmethod
        def main(argv):
            Fake.argv = argv
            return 0

    assert dev_cli.main(["bench", "--device", "tpu"], cli_module=Fake) == 2
    assert dev_cli.main(["bench", "--device=cpu", "--trials", "2"], cli_module=Fake) == 0
    assert Fake.argv == ["bench", "--trials", "2"] and Fake._run_estimator is None
    assert dev_cli.main(["separate", "--device", "cuda", "--iterations", "3"], cli_module=Fake) == 0
    assert Fake.argv == ["separate", "--iterations", "3"] and Fake._run_estimator is dev_cli.run_estimator


def test_lazy_statistics_fields_materialise_once():
    # TransformedStats / PosteriorStats hold device tensors until first read (paper_1805_09498_b200/_lazy.py)
    import dataclasses
    import pickle

    from paper_1805_09498_b200._lazy import DeviceArray
    from paper_1805_09498_b200.fastfca import TransformedStats
    from paper_1805_09498_b200.fca import PosteriorStats

    class FakeTensor:  # stands in for a CUDA tensor: .cpu().numpy()
        copies = 0

        def __init__(self, a):
            self.a = a

        def cpu(self):
            FakeTensor.copies += 1
            return self

        def numpy(self):
            return self.a

    for cls in (TransformedStats, PosteriorStats):
        FakeTensor.copies = 0
        mu, phi = np.arange(6.0).reshape(2, 3) + 1j, np.ones((2, 3))
        st = cls(mu=DeviceArray(FakeTensor(mu)), phi=DeviceArray(FakeTensor(phi)))
        assert st.device_tensor("mu") is not None and FakeTensor.copies == 0
        assert np.array_equal(st.mu, mu) and np.array_equal(st.mu, mu) and FakeTensor.copies == 1
        assert st.device_tensor("mu") is None and st.device_tensor("phi") is not None
        d = dataclasses.asdict(st)  # reads phi too
        assert FakeTensor.copies == 2 and np.array_equal(d["phi"], phi)
        rep = dataclasses.replace(st, phi=np.zeros((2, 3)))
        assert isinstance(rep.mu, np.ndarray) and not rep.phi.any()
        back = pickle.loads(pickle.dumps(st))
        assert np.array_equal(back.mu, mu) and np.array_equal(back.phi, phi)
        assert [f.name for f in dataclasses.fields(cls)] == ["mu", "phi"]
