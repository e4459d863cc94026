"""Device switch for the reference's command-line driver (``fcasep.cli``), SURVEY.md §8(f) #3.

``fcasep.cli`` runs every estimator call through two module-level hooks,
``_run_estimator`` (cli.py:202-208) and ``_images_from_run`` (cli.py:211-214);
``separate_once`` (cli.py:217-260) and ``cmd_bench`` (cli.py:292-389) look them
up at call time.  ``install(cli_module)`` rebinds both hooks to the B200 path,
so ``separate`` and ``bench`` -- scene synthesis, WAV I/O, SDR, the CSV report
and the manifest unchanged -- time and run the estimator and the Wiener images
on the device.  ``main(argv)`` is the reference CLI with one extra option,
``--device {cpu,cuda}`` (default cuda):

    python -m paper_1805_09498_b200.cli bench --trials 2 --iterations 20 --device cuda

The reference package itself is the caller here (it is not part of this
package); its objects are converted at the boundary: ``obs.data`` (I, N, F) and
the parameter arrays go in as they are, and the results come back as this
package's run / image types, which carry the reference's field names
(params, stats, counters with ``as_dict``; images with ``stft``).
"""

from __future__ import annotations

import sys

from . import fastfca, fca, wiener
from .stft import ObservationTensor


def _obs(obs) -> ObservationTensor:
    return obs if isinstance(obs, ObservationTensor) else ObservationTensor(obs.data, check_finite=False)


def run_estimator(cfg, obs, params, record_likelihood: bool = False):
    """``cli._run_estimator`` (cli.py:202-208) on the device."""
    o = _obs(obs)
    if cfg.algorithm == "fca":
        init = params if isinstance(params, fca.FcaParams) else fca.FcaParams(S=params.S, v=params.v)
        return fca.run_fca(o, init, cfg.iterations, record_likelihood=record_likelihood)
    init = (params if isinstance(params, fastfca.FastFcaParams)
            else fastfca.FastFcaParams(P=params.P, Lam=params.Lam, v=params.v))
    return fastfca.run_fastfca(o, init, cfg.iterations, cfg.inner_k, record_likelihood=record_likelihood)


def images_from_run(cfg, run, obs):
    """``cli._images_from_run`` (cli.py:211-214) on the device: (J, I, N, F) source images."""
    if cfg.algorithm == "fca":
        return wiener.mmse_images_fca(run.params, _obs(obs))
    return wiener.mmse_images_fastfca(run.params, run.stats)


def install(cli_module) -> None:
    """Route a reference CLI module's estimator and image hooks through the device path."""
    cli_module._run_estimator = run_estimator
    cli_module._images_from_run = images_from_run


def main(argv=None, cli_module=None) -> int:
    """The reference CLI (``fcasep.cli.main``) with ``--device {cpu,cuda}``."""
    argv = list(sys.argv[1:] if argv is None else argv)
    device = "cuda"
    for k, a in enumerate(argv):
        if a == "--device" and k + 1 < len(argv):
            device = argv[k + 1]
            del argv[k:k + 2]
            break
        if a.startswith("--device="):
            device = a.split("=", 1)[1]
            del argv[k]
            break
    if device not in ("cpu", "cuda"):
        print(f"error: --device must be cpu or cuda, got {device!r}", file=sys.stderr)
        return 2
    if cli_module is None:
        from fcasep import cli as cli_module  # the reference package drives the CLI
    if device == "cuda":
        install(cli_module)
    return cli_module.main(argv)


if __name__ == "__main__":
    sys.exit(main())
