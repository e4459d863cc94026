"""CPU oracle for the FastFCA-AS hot path -- TEST INFRASTRUCTURE ONLY.

This package is a plain-numpy restatement of the reference algorithm
(``/root/reference/pkg/src/fcasep``) used as the *checker* for the CUDA
path.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs (as the fallback when the stock
reference is not installed in ``baseline/_ref``) and its after-the-timed-region
parity check of the timed batch may import it -- always as the checker, never
as the thing measured.  The product
package ``paper_1805_09498_b200`` never imports anything from here and has no
CPU fallback.

Parity pin: ``tests/test_oracle_golden.py`` checks every function here
against golden vectors produced by running the unmodified reference in the
build container (``tests/golden/make_golden.py``).

All arithmetic is float64 / complex128 (the reference has no 32-bit path,
``SPEC.md:146``); the complex64 oracle is this code on exactly-upcast inputs.
"""

from . import fastfca_ref, fca_ref, pipeline_ref, scene_ref, stft_ref  # noqa: F401
