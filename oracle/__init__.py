"""FP64 CPU oracle for windowed root-MUSIC fringe demodulation (arxiv 1910.11872).

TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import anything from here.
The product path (``paper_1910_11872_b200``) never imports this package, and this package
never imports the product path: the two share no code.
"""

from .rootmusic import (  # noqa: F401
    FLAG_AMBIGUOUS,
    FLAG_BORDER,
    FLAG_LOW_AMPLITUDE,
    FLAG_NONCONVERGED,
    FLAG_NONFINITE,
    FLAG_SMALL_GAP,
    PARITY_EXCLUDE_MASK,
    companion_roots,
    demod_frame,
    demod_stack,
    estimate_windows,
    extract_windows,
    index_gradient,
    vertical_profile,
    music_polynomial,
    noise_projectors,
    select_root,
    svd_subspaces,
    window_offsets,
    wrap,
)
from .analytic import analytic_signal, lobe_mask  # noqa: E402,F401
from . import unwrap  # noqa: E402,F401
