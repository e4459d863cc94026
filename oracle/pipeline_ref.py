"""CPU restatement of the reference's in-memory separation pipeline -- TEST INFRASTRUCTURE ONLY.

Chains the oracle restatements the way ``cli.separate_once`` (cli.py:217-260)
chains the reference modules: analyze (stft.py:96-112) -> init
(scene.py:250-271) -> estimator (fastfca.py:401-474 / fca.py:187-215) ->
Wiener images (wiener.py:32-43) -> resynthesis (wiener.py:46-53) -> SDR
(evalkit.py:68-88).  Pinned against the reference's own output in
tests/golden/golden.npz (``pipe/*``).
"""

from __future__ import annotations

import numpy as np

from . import fastfca_ref, fca_ref, scene_ref, stft_ref

SDR_CAP_DB = 200.0  # evalkit.py:23


def compute_sdr(reference, estimate) -> float:
    """evalkit.py:68-88."""
    ref_energy = float(np.sum(reference ** 2))
    err_energy = float(np.sum((reference - estimate) ** 2))
    if err_energy < 1e-20 * ref_energy:
        return SDR_CAP_DB
    return float(10.0 * np.log10(ref_energy / err_energy))


def separate_once(mixture, references, algorithm="fastfca", init="oracle", sources=3, iterations=20,
                  inner_k=1, seed=0, L=1024, shift=512):
    """Returns (audio (J, I, S_out), sdr list, final params tuple)."""
    y = stft_ref.analyze(mixture, L, shift)
    if init == "oracle":
        X = np.stack([stft_ref.analyze(r, L, shift) for r in references])
        S_hat, v_hat = scene_ref.oracle_covariances(X, y)
    else:
        S_hat, v_hat = scene_ref.diffuse_covariances(y, sources, seed)
    if algorithm == "fastfca":
        P0, lam0, v0 = fastfca_ref.params_from_covariances(S_hat, v_hat)
        run = fastfca_ref.run_fastfca(y, P0, lam0, v0, iterations, inner_k)
        imgs = fastfca_ref.images(run.P, run.mu)
        params = (run.P, run.lam, run.v)
    else:
        run = fca_ref.run_fca(y, S_hat, v_hat, iterations)
        mu, _ = fca_ref.e_step(run.S, run.v, y)
        imgs = mu.transpose(0, 3, 1, 2)
        params = (run.S, run.v)
    J, I, N, F = imgs.shape
    audio = stft_ref.synthesize(imgs.reshape(J * I, N, F), L, shift).reshape(J, I, -1)
    sdrs = []
    if references is not None:
        for j in range(references.shape[0]):
            n = min(references.shape[2], audio.shape[2])
            sdrs.append(compute_sdr(references[j, :, :n], audio[j, :, :n]))
    return audio, sdrs, params
