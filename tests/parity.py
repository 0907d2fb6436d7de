"""Shared parity helpers: compare CUDA-path outputs with the oracle under the
acceptance procedure of DESIGN.md §3:

  1. expected: shift equal, f_min bit-equal (u16) / within 1e-4 relative (f32),
     corrected frame bit-equal;
  2. float32 only: otherwise the GPU shift must be one the oracle reaches by
     taking a near-tie winner (best two f within 1e-4 relative) at some level, with
     f_min within 1e-4 of the oracle's f there and the corrected frame equal
     to the oracle's apply_shift with that shift.
"""
import numpy as np

import oracle

FMIN_REL = 1e-4   # BASELINE.json north_star: "f_min must agree within 1e-4 relative"


def check_frame(frame, template, w, levels, shift, fmin, corrected=None, exact=True):
    """Returns 'exact' or 'near-tie'; raises AssertionError otherwise.

    ``exact=True`` (uint16 input) demands the oracle's own shift and a bit-equal
    f_min: every N is computed exactly on both sides, so any
    other shift is a bug and the near-tie exemption never applies."""
    r = oracle.align_frame(frame, template, w, levels)
    s, t = int(shift[0]), int(shift[1])
    if exact:
        assert (s, t) == (r.s, r.t), f"shift {(s, t)} != oracle {(r.s, r.t)} (u16: must be exact)"
    if (s, t) == (r.s, r.t):
        if exact:
            assert float(fmin) == r.fmin, f"fmin {fmin!r} != oracle {r.fmin!r}"
        else:
            assert abs(float(fmin) - r.fmin) <= FMIN_REL * abs(r.fmin) + 1e-300
        kind = "exact"
        ref_f = r.fmin
    else:
        acc = oracle.acceptable_results(frame, template, w, levels)
        assert (s, t) in acc, f"shift {(s, t)} not acceptable; oracle {(r.s, r.t)} near-ties {list(acc)}"
        ref_f = acc[(s, t)]
        assert abs(float(fmin) - ref_f) <= FMIN_REL * abs(ref_f) + 1e-300
        kind = "near-tie"
    if corrected is not None:
        assert np.array_equal(np.asarray(corrected), oracle.apply_shift(frame, s, t)), "corrected frame differs"
    return kind
