"""CPU oracle for moco (TEST INFRASTRUCTURE ONLY -- see moco_oracle.py header).

Importable only from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  Shares no code with the CUDA path.
"""
from .moco_oracle import *  # noqa: F401,F403
from .moco_oracle import (NEAR_TIE_REL, FrameResult, LevelResult, acceptable_results,  # noqa: F401
                          align_frame, align_stack, apply_shift, area, coarse_search,
                          downsample, objective, objective_grid, overlap, pyramid,
                          refine, select, sum_sq_diff)
