"""Command line: ``python -m paper_1506_06039_b200.cli align|synth ...`` (SURVEY.md
section 8(f-4); the CLI shape follows SPEC.md:423-435, the defaults).

  align --input STACK --output STACK [--template-index N | --template-file STACK]
        [--max-shift N|auto] [--levels 0|1|2|auto] [--bits 12] [--shifts-csv PATH]
        [--mean-before PATH] [--mean-after PATH] [--algo auto|tc|fft|direct]
  synth --config K [--frames T] --output STACK [--truth-csv PATH]

Every step of the alignment runs on the GPU through the C-ABI (Plan); this module only
moves files.  Exit 0 on success, 2 on invalid input (usage on stderr).
"""
from __future__ import annotations

import argparse
import sys

import numpy as np


def _parser():
    ap = argparse.ArgumentParser(prog="moco")
    sub = ap.add_subparsers(dest="cmd", required=True)
    a = sub.add_parser("align")
    a.add_argument("--input", required=True)
    a.add_argument("--output", required=True)
    g = a.add_mutually_exclusive_group()
    g.add_argument("--template-index", type=int, default=0)
    g.add_argument("--template-file")
    a.add_argument("--max-shift", default="auto", help="w at the coarsest level, or auto (P:49)")
    a.add_argument("--levels", default="auto", help="0, 1, 2 or auto (P:49)")
    a.add_argument("--bits", type=int, default=None, help="sample bit depth (default: from the data)")
    a.add_argument("--shifts-csv")
    a.add_argument("--mean-before")
    a.add_argument("--mean-after")
    a.add_argument("--algo", default="auto", choices=["auto", "tc", "fft", "direct"])
    a.add_argument("--device", type=int, default=0)
    s = sub.add_parser("synth")
    s.add_argument("--config", type=int, required=True)
    s.add_argument("--frames", type=int, default=None)
    s.add_argument("--output", required=True)
    s.add_argument("--truth-csv")
    return ap


def align_cmd(args) -> int:
    import torch

    from . import io
    from ._lib import Plan, auto_config
    stack = io.load_stack(args.input)
    T, m, n = stack.shape
    if stack.dtype == np.uint8:
        stack = stack.astype(np.uint16)
    if args.template_file:
        tpl = io.load_stack(args.template_file)[0].astype(np.uint16)
    else:
        if not 0 <= args.template_index < T:
            print(f"moco: --template-index {args.template_index} outside the stack (T={T})", file=sys.stderr)
            return 2
        tpl = stack[args.template_index]
    w_auto, l_auto = auto_config(m, n)
    levels = l_auto if args.levels == "auto" else int(args.levels)
    if levels not in (0, 1, 2):
        print("moco: --levels must be 0, 1 or 2 (PAPER.md:49: downsampling 3 and 4 times causes "
              "severe errors)", file=sys.stderr)
        return 2
    w = min(m >> levels, n >> levels) // 3 if args.max_shift == "auto" else int(args.max_shift)
    if args.max_shift == "auto" and args.levels == "auto":
        w = w_auto
    bits = args.bits or max(1, int(stack.max()).bit_length())
    bits = min(bits, 16 - 2 * levels)
    dev = torch.device("cuda", args.device)
    frames = torch.from_numpy(stack).to(dev)
    plan = Plan(m, n, w, levels, "u16", bits, device=args.device, algo=None if args.algo == "auto" else args.algo)
    plan.set_template(torch.from_numpy(np.ascontiguousarray(tpl)).to(dev))
    sh, fm, co, fl = plan.align(frames, corrected=True, flags=True)
    torch.cuda.synchronize()
    io.save_stack(co.cpu().numpy(), args.output)
    if args.shifts_csv:
        io.write_shift_log(args.shifts_csv, sh.cpu().numpy(), fm.cpu().numpy(), fl.cpu().numpy())
    if args.mean_before:
        io.save_stack(io.mean_image(frames).cpu().numpy(), args.mean_before)
    if args.mean_after:
        io.save_stack(io.mean_image(co).cpu().numpy(), args.mean_after)
    print(f"moco: aligned {T} frames of {m}x{n} (w={w}, levels={levels}, algo={plan.algo})", file=sys.stderr)
    return 0


def synth_cmd(args) -> int:
    from synth import config_spec, make_stack

    from . import io
    spec = config_spec(args.config, **({"T": args.frames} if args.frames else {}))
    st = make_stack(spec, 0, spec.T)
    fr = st.frames.numpy()
    if fr.dtype != np.uint16:
        print("moco: synth writes 16-bit stacks only (config 0 is float32)", file=sys.stderr)
        return 2
    io.save_stack(fr, args.output)
    if args.truth_csv:
        with open(args.truth_csv, "w") as f:
            f.write("frame,dy,dx,stripe\n")
            for k in range(len(fr)):
                f.write(f"{k},{int(st.shifts[k, 0])},{int(st.shifts[k, 1])},{int(st.stripe[k])}\n")
    return 0


def main(argv=None) -> int:
    try:
        args = _parser().parse_args(argv)
    except SystemExit as e:
        return 2 if e.code else 0
    try:
        return align_cmd(args) if args.cmd == "align" else synth_cmd(args)
    except (ValueError, OSError) as e:
        print(f"moco: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
