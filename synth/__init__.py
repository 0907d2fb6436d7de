"""Seeded synthetic calcium-imaging stacks shaped like BASELINE.json's configs.

This module holds NONE of moco's arithmetic (no objective, no search, no
pyramid): it only draws inputs.  Both sides of every parity check -- the CPU
oracle (``oracle/``) and the CUDA path (``paper_1506_06039_b200``) -- are fed
the same bytes produced here.  The recipe is SURVEY.md §8(d) and is restated
in DESIGN.md §4.
"""
from .generator import CONFIGS, ConfigSpec, Stack, make_stack, config_spec  # noqa: F401
