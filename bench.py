#!/usr/bin/env python
"""bench.py -- frames/s of the moco hot path on B200 (BASELINE.json metric).

Default workload: BASELINE.json configs[2] ("C2"): 10,000 frames of 512x512
uint16 (12-bit), one 2x2 level to 256x256, w=16 there, +-1 refine at 512x512,
corrected frames written.  A step = one moco_align_batch over the whole
(per-rank) stack: every step of the hot path (S1..S7) on every frame.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl moco|reference]

N>1 is launched by torch.distributed.run (one rank per GPU, NCCL): weak
scaling -- every rank aligns its own contiguous 10,000-frame block of an
N*10,000-frame stack, the template is broadcast from rank 0 (setup), and each timed
step ends with an NCCL all_gather of the per-frame results (shifts, f_min) -- or, with
``--gather peer``, the library's kernels store every frame's record straight into rank
0's memory over NVLink (CUDA symmetric memory, one device-side barrier per step); timing
is the max over ranks of CUDA-event time.

Rank 0 prints ONE JSON line (contract in the task statement / DESIGN.md §8).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth import config_spec, make_stack  # noqa: E402

METRIC = "frames/sec aligned (512x512 uint16, w=16)"
UNIT = "frames/s"


def read_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return {"hbm_gbs": float(d["hbm_gbs"]), "bf16_tflops": float(d["bf16_tflops"]),
                "sm_max_mhz": float(d.get("sm_max_mhz", 1965.0)), "source": "measured"}
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0, "source": "fallback"}


# ----------------------------------------------------------------- work models
def fft_model(spec):
    """SURVEY.md §8(d) minimal algorithmic FLOPs per frame (the roofline model
    of BASELINE.md §2): FFT correlation + energy + score + downsample + refine."""
    L = spec.levels
    mc, nc = spec.m >> L, spec.n >> L
    P = (mc + spec.w) * (nc + spec.w)
    W = 2 * spec.w - 1
    f_fft = 2 * 2.5 * P * math.log2(P) + 3 * P
    f_energy = 2 * mc * nc
    f_score = 6 * W * W
    f_down = 0.75 * sum((spec.m >> l) * (spec.n >> l) for l in range(L))
    f_refine = sum(20 * (spec.m >> l) * (spec.n >> l) for l in range(L))
    return {"coarse": f_fft + f_energy + f_score, "downsample": f_down, "refine": f_refine,
            "total": f_fft + f_energy + f_score + f_down + f_refine}


def kernel_models(spec, esz, algo):
    """Per-frame algorithmic work of each kernel kind -> (bound, amount, unit)."""
    L = spec.levels
    m, n = spec.m, spec.n
    mc, nc = m >> L, n >> L
    W = 2 * spec.w - 1
    fm = fft_model(spec)
    down_bytes = sum((m >> l) * (n >> l) * esz + (m >> (l + 1)) * (n >> (l + 1)) * 2 for l in range(L))
    if algo == "tc":
        # exact int8 direct correlation: 4 part products (hi/lo x hi/lo) per pixel per lag
        coarse = ("tensor_i8", 2.0 * 4 * W * W * mc * nc, "op")
        prep = ("hbm", m * n * esz + 2 * (mc + 64) * nc, "B")
    elif algo == "fft":
        # kernels_fft2.cuh: rows (block sums, energies, forward row FFTs) = MOCO_K_PREP, columns
        # (forward column FFTs, spectrum product, inverse column FFTs) = MOCO_K_COARSE, score
        # (inverse row FFTs of the lag rows, certified intervals) = MOCO_K_SCORE; the
        # SURVEY §8(d) FFT flops split 1/4 : 1/2 + product : 1/4
        P_ = (mc + spec.w) * (nc + spec.w)
        half = 2.5 * P_ * math.log2(P_)
        coarse = ("alu", half + 3 * P_, "flop")
        prep = ("alu", 0.5 * half + 2 * mc * nc, "flop")
    else:
        coarse = ("alu", 2.0 * W * W * mc * nc, "op")
        prep = ("hbm", mc * nc * 2, "B")
    return {
        "downsample": ("hbm", down_bytes, "B"),
        "coarse": coarse,
        "tc_prep": prep,
        "tc_score": ("alu", (0.5 * 2.5 * (mc + spec.w) * (nc + spec.w) * math.log2((mc + spec.w) * (nc + spec.w))
                             if algo == "fft" else 0) + 6 * W * W, "flop"),
        # tensor-core refine sums (kernels_rtc.cuh): one read of each refine level's frame;
        # the MMAs need < 10 % of the tensor pipe, so the bound is the read
        "refine": ("hbm", sum((m >> l) * (n >> l) * 2 for l in range(L)), "B") if esz == 2
        else ("alu", fm["refine"], "flop"),
        "apply": ("hbm", 2 * m * n * esz, "B"),
    }


# ---------------------------------------------------------------- clock sampler
class ClockSampler:
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "50",
                 "-i", str(self.index)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()   # nvidia-smi can take seconds to start on a fresh box
            while not self.lines and time.time() - t0 < 15 and self.proc.poll() is None:
                time.sleep(0.02)
        except Exception:
            self.proc = None
        self.i0 = 0

    def mark(self):
        """Start of the timed region: samples before it are dropped."""
        self.i0 = len(self.lines)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        # the samples taken during the timed region (at least the first one after it)
        for ln in self.lines[self.i0:] or self.lines[-1:]:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(max(smax)) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------- CPU oracle
def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def cpu_oracle_rate(frames_np, template_np, spec, nframes):
    import oracle
    cores = len(os.sched_getaffinity(0))
    sel = frames_np[:nframes]
    t0 = time.perf_counter()
    oracle.align_stack(sel, template_np, spec.w, spec.levels, workers=cores)
    dt = time.perf_counter() - t0
    return len(sel) / dt, cores, dt


def parity_report(frames, template, shifts, fmin, corrected, spec, budget_s=25.0, stride=10):
    """The oracle (fp64, brute force, process pool over the host cores) on every `stride`-th
    frame of the timed workload -- up to what the host finishes in about `budget_s` --
    against the GPU results of the timed steps: counts of exact / near-tie / failed frames
    (uint16: only exact counts, any other shift is a failure; SURVEY.md section 8(c)
    acceptance), corrected frames compared bit for bit on the first 32 sampled frames.
    The same run gives the oracle's frames/s (cpu_baseline)."""
    import oracle
    cores = len(os.sched_getaffinity(0))
    tp = template.cpu().numpy()
    T = frames.shape[0]
    # pilot: rate on a small sample sizes the parity sample to the time budget
    def take(x, idx):   # (integer-array indexing is not implemented for uint16 on CUDA)
        y = x.view(torch.int16) if x.dtype == torch.uint16 else x
        y = y[torch.as_tensor(idx, device=x.device)].cpu()
        return (y.view(torch.uint16) if x.dtype == torch.uint16 else y).numpy()

    pilot = list(range(0, min(T, 10 * cores), 10))[: max(4, cores)]
    t0 = time.perf_counter()
    oracle.align_stack(take(frames, pilot), tp, spec.w, spec.levels, workers=cores)
    rate0 = len(pilot) / (time.perf_counter() - t0)
    want = max(len(pilot), int(rate0 * budget_s))
    idx = list(range(0, T, stride))
    if len(idx) > want:
        idx = idx[:: int(math.ceil(len(idx) / want))]
    fr = take(frames, idx)
    t0 = time.perf_counter()
    osh, ofm = oracle.align_stack(fr, tp, spec.w, spec.levels, workers=cores)
    dt = time.perf_counter() - t0
    sh = take(shifts, idx)
    fm = take(fmin, idx)
    exact = near = failed = 0
    bad = []
    for j, k in enumerate(idx):
        same = tuple(sh[j]) == tuple(osh[j])
        if spec.dtype == "u16":
            ok = same and fm[j] == ofm[j]
            exact += ok
            if not ok:
                failed += 1
                bad.append(k)
        elif same and abs(fm[j] - ofm[j]) <= 1e-4 * abs(ofm[j]):
            exact += 1
        else:
            acc = oracle.acceptable_results(fr[j], tp, spec.w, spec.levels)
            key = (int(sh[j, 0]), int(sh[j, 1]))
            if key in acc and abs(fm[j] - acc[key]) <= 1e-4 * abs(acc[key]):
                near += 1
            else:
                failed += 1
                bad.append(k)
    co_bad = 0
    for j, k in enumerate(idx[:32]):
        if not np.array_equal(corrected[k].cpu().numpy(), oracle.apply_shift(fr[j], int(osh[j, 0]), int(osh[j, 1]))):
            co_bad += 1
    step_ = idx[1] - idx[0] if len(idx) > 1 else 1
    return {"frames_checked": len(idx), "sample": f"every {step_}-th frame of the {T}-frame timed stack",
            "exact": int(exact), "near_tie": int(near), "failed": int(failed), "failed_frames": bad[:16],
            "corrected_checked": min(32, len(idx)), "corrected_failed": co_bad,
            "oracle_fps": len(idx) / dt, "oracle_s": dt, "cores": cores, "cpu_model": cpu_model()}


def reference_arm(args, spec, rank, world):
    """--impl reference: the CPU oracle (the reference for this tier), timed on
    the host cores on bounded samples of the same workload."""
    if rank != 0:
        return
    import oracle
    from concurrent.futures import ProcessPoolExecutor
    cores = len(os.sched_getaffinity(0))
    per_step = max(1, min(cores, 64))
    need = per_step * (args.steps + args.warmup)
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    st = make_stack(spec, 0, min(spec.T, need), device=dev)
    fr = st.frames.cpu().numpy()
    tp = st.template.cpu().numpy()
    ex = ProcessPoolExecutor(max_workers=cores)
    jobs = lambda k: [(fr[(k * per_step + i) % len(fr)], tp, spec.w, spec.levels) for i in range(per_step)]
    for k in range(args.warmup):
        list(ex.map(oracle.moco_oracle._align_one, jobs(k)))
    t0 = time.perf_counter()
    for k in range(args.steps):
        list(ex.map(oracle.moco_oracle._align_one, jobs(args.warmup + k)))
    dt = time.perf_counter() - t0
    ex.shutdown()
    value = per_step * args.steps / dt
    sample = f"{per_step} frames/step of config {spec.index} (of {spec.T}), oracle fp64 numpy, process pool"
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "config": workload_config(spec, world, None),
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def gpu_local_cpus(dev):
    """The host CPUs NVML reports as local to `dev` (its NUMA node), or None."""
    try:
        import pynvml
        pr = torch.cuda.get_device_properties(dev)
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByPciBusId(f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0")
        n = os.cpu_count() or 1
        mask = pynvml.nvmlDeviceGetCpuAffinity(h, (n + 63) // 64)
        cpus = {i for i in range(n) if (mask[i // 64] >> (i % 64)) & 1} & os.sched_getaffinity(0)
        return cpus or None
    except Exception:
        return None


def pinned_ceiling(hf, hc, dev, nbytes=256 << 20):
    """Frames/s the PCIe link allows through THESE pinned buffers: H2D from hf and D2H into
    hc at once on two streams (frame in + corrected out per frame), timed with events."""
    try:
        a8, c8 = hf.view(-1).view(torch.uint8), hc.view(-1).view(torch.uint8)
        n = min(nbytes, a8.numel(), c8.numel())
        d_in = torch.empty(n, dtype=torch.uint8, device=dev)
        d_out = torch.empty(n, dtype=torch.uint8, device=dev)
        s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        cur = torch.cuda.current_stream(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for it in range(2):
            e0.record(cur)
            s1.wait_stream(cur)
            s2.wait_stream(cur)
            for _ in range(4):
                with torch.cuda.stream(s1):
                    d_in.copy_(a8[:n], non_blocking=True)
                with torch.cuda.stream(s2):
                    c8[:n].copy_(d_out, non_blocking=True)
            cur.wait_stream(s1)
            cur.wait_stream(s2)
            e1.record(cur)
        torch.cuda.synchronize(dev)
        dt = e0.elapsed_time(e1) / 1e3 / 4
        gbs = n / dt / 1e9
        fbytes = hf[0].numel() * hf.element_size()
        return {"bidir_each_GBps": gbs, "ceiling_fps": gbs * 1e9 / fbytes}
    except Exception as e:
        return {"error": str(e)[:120]}


def workload_config(spec, world, algo):
    L = spec.levels
    return {"workload": f"C{spec.index}: {spec.T} frames/rank of {spec.m}x{spec.n} "
                        f"{'uint16 12-bit' if spec.dtype == 'u16' else 'float32'}, levels={L}, "
                        f"w={spec.w} at {spec.m >> L}x{spec.n >> L}, corrected frames written",
            "config_index": spec.index, "frames_per_rank": spec.T, "m": spec.m, "n": spec.n,
            "levels": L, "w": spec.w, "coarse_algo": algo,
            "l2": "no flush needed: per-step input %.2f GB > 126 MB L2" % (spec.T * spec.m * spec.n * (2 if spec.dtype == 'u16' else 4) / 1e9),
            "parallelism": f"dp{world} (frame blocks)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)   # ~0.22 s timed: several 50-ms clock samples
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--frames", type=int, default=None, help="override frames per rank")
    ap.add_argument("--impl", default="moco", choices=["moco", "reference"])
    ap.add_argument("--algo", default="auto", choices=["auto", "direct", "tc", "fft"])
    ap.add_argument("--gather", default="nccl", choices=["peer", "nccl"],
                    help="N>1: per-frame results by an NCCL all-gather (default: the path that has run "
                         "at N>1), or stored into rank 0's memory by the kernels over peer memory (fused; "
                         "tested at N=1 only)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-paper", action="store_true", help="skip the paper-default (w=85) context line")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "moco" else args.warmup

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    spec = config_spec(args.config)
    if args.frames:
        spec = config_spec(args.config, T=args.frames)

    if args.impl == "reference":
        return reference_arm(args, spec, rank, world)

    import torch.distributed as dist
    from paper_1506_06039_b200 import Plan
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    # per-rank block of an (N * T)-frame stack (weak scaling); chunk-seeded so
    # every rank regenerates exactly its own frames
    Tl = spec.T
    full = config_spec(spec.index, T=Tl * world)
    st = make_stack(full, rank * Tl, Tl, device=dev)
    frames = st.frames
    template = st.template
    if world > 1:   # template from rank 0 over NCCL (plan setup, untimed)
        from paper_1506_06039_b200.dist import broadcast_template
        broadcast_template(template, src=0)
    esz = frames.element_size()
    plan = Plan(spec.m, spec.n, spec.w, spec.levels, spec.dtype, 12, device=local)
    if args.algo != "auto":
        plan.set_algo(args.algo)
    plan.set_template(template)
    shifts = torch.empty((Tl, 2), dtype=torch.int32, device=dev)
    fmin = torch.empty((Tl,), dtype=torch.float64, device=dev)
    corrected = torch.empty_like(frames)
    from paper_1506_06039_b200.dist import PeerResults, gather_results
    peer = None
    gather_mode = None
    if world > 1:
        gather_mode = args.gather
        if args.gather == "peer":
            try:   # fused: the kernels store each frame's record into rank 0's memory
                peer = PeerResults(Tl, dev)
            except Exception as e:   # (no symmetric memory on this node: the NCCL all-gather)
                print(f"[bench] peer-memory gather unavailable ({str(e)[:120]}); NCCL all-gather", file=sys.stderr)
                gather_mode = "nccl"
            ok = torch.tensor([1 if peer is not None else 0], dtype=torch.int32, device=dev)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)   # every rank takes the same path
            if int(ok.item()) == 0:
                peer, gather_mode = None, "nccl"

    def step():
        if peer is not None:
            plan.align_into(frames, peer.shifts, peer.fmin, corrected)
            peer.barrier()
            return
        plan.align_into(frames, shifts, fmin, corrected)
        if world > 1:   # per-frame results of every rank to every rank (16 B/frame)
            gather_results(shifts, fmin, world * Tl)

    for _ in range(args.warmup):
        step()
    launches_per_step = plan.launches
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.3)
    plan.profile(True)
    plan.profile_read()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    clk.mark()
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    prof = plan.profile_read()
    plan.profile(False)
    clocks = clk.stop()
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    ms_step = ms / args.steps
    value = world * Tl / (ms_step / 1e3)

    # ---- roofline of the dominant kernel (largest share of the timed region)
    peaks = read_peaks()
    models = kernel_models(spec, esz, plan.algo)
    kind = max((k for k in prof if prof[k][1] > 0), key=lambda k: prof[k][0])
    kms, klaunch = prof[kind]
    frames_timed = Tl * args.steps
    bound, per_frame, _u = models[kind]
    if bound == "hbm":
        achieved = per_frame * frames_timed / (kms / 1e3) / 1e9
        peak, unit = peaks["hbm_gbs"], "GB/s"
        peak_note = f"MEASURED_PEAKS.json hbm_gbs ({peaks['source']})"
    elif bound == "tensor_i8":
        bound = "tensor"
        achieved = per_frame * frames_timed / (kms / 1e3) / 1e12
        peak, unit = 2.0 * peaks["bf16_tflops"], "TOP/s"
        peak_note = (f"int8 dense = 2 x MEASURED_PEAKS.json bf16_tflops burst ({peaks['source']}; "
                     "B200 nominal int8:bf16 = 4.5:2.25 P)")
    else:
        achieved = per_frame * frames_timed / (kms / 1e3) / 1e12
        peak = 148 * 128 * 2 * peaks["sm_max_mhz"] * 1e6 / 1e12
        unit = "TFLOP/s"
        peak_note = "148 SM x 128 FP32/INT32 lanes x 2 x sm_max_mhz (DESIGN.md §8)"
    traffic = None
    isolated = None
    try:
        ncu = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        entry = ncu.get(f"C{spec.index}", {}).get(plan.algo, {}).get(kind)
        if entry:   # per-frame DRAM bytes from the committed ncu capture x frames per launch
            traffic = entry["bytes_per_frame"] * frames_timed / klaunch
            # the same kernel alone (ncu, serialised launches): the live duration above
            # includes the time it shares the GPU with the other two pipeline streams
            us = entry["duration_us"] / entry["frames_in_capture"]
            ach = per_frame / (us * 1e-6) / (1e9 if bound == "hbm" else 1e12)
            isolated = {"us_per_frame": us, "achieved": ach, "frac": ach / peak,
                        "source": "profiles/ncu_traffic.json (ncu --set full, one launch alone)"}
    except Exception:
        pass
    roofline = {"bound": bound, "achieved": achieved, "peak": peak, "unit": unit,
                "frac": achieved / peak, "traffic": traffic, "kernel": kind, "isolated": isolated,
                "kernel_share": kms / ms if ms > 0 else None,
                "per_frame_work": per_frame, "peak_source": peak_note,
                "kernels_ms": {k: round(v[0], 4) for k, v in prof.items() if v[1]},
                "kernels_launches": {k: v[1] for k, v in prof.items() if v[1]}}
    fm = fft_model(spec)
    hbm_roof_fps = peaks["hbm_gbs"] * 1e9 / (2 * spec.m * spec.n * esz)
    alu_roof_fps = 148 * 128 * 2 * peaks["sm_max_mhz"] * 1e6 / fm["total"]
    step_roof = min(hbm_roof_fps, alu_roof_fps)

    # ---- single-frame latency (closed-loop use case), device-resident frame
    lat = None
    if rank == 0:
        one = frames[:1]
        s1, f1, c1 = shifts[:1], fmin[:1], corrected[:1]
        for _ in range(20):
            plan.align_into(one, s1, f1, c1)
        ts = []
        for _ in range(200):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            plan.align_into(one, s1, f1, c1)
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b))
        lat = {"p50_ms": float(np.percentile(ts, 50)), "p99_ms": float(np.percentile(ts, 99))}
        # host wall time, call -> results on the device and the stream drained
        hs = []
        for _ in range(200):
            t0 = time.perf_counter()
            plan.align_into(one, s1, f1, c1)
            torch.cuda.current_stream().synchronize()
            hs.append((time.perf_counter() - t0) * 1e3)
        lat.update(host_p50_ms=float(np.percentile(hs, 50)), host_p99_ms=float(np.percentile(hs, 99)))
        # the same call captured once in a CUDA graph and replayed (launch overhead removed)
        try:
            g = torch.cuda.CUDAGraph()
            cs = torch.cuda.Stream()
            cs.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(cs):
                plan.align_into(one, s1, f1, c1)   # warm on the capture stream
                torch.cuda.synchronize()
                with torch.cuda.graph(g, stream=cs):
                    plan.align_into(one, s1, f1, c1)
            torch.cuda.synchronize()
            # reference from a separate direct call, then a sentinel in the outputs: the
            # replays must rewrite them (a replay that did nothing would leave -1)
            plan.align_into(one, s1, f1, c1)
            torch.cuda.synchronize()
            ref = s1.clone()
            s1.fill_(-1)
            ge, gh = [], []
            for _ in range(200):
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                t0 = time.perf_counter()
                a.record()
                g.replay()
                b.record()
                b.synchronize()
                gh.append((time.perf_counter() - t0) * 1e3)
                ge.append(a.elapsed_time(b))
            lat["graph"] = {"p50_ms": float(np.percentile(ge, 50)), "p99_ms": float(np.percentile(ge, 99)),
                            "host_p50_ms": float(np.percentile(gh, 50)), "host_p99_ms": float(np.percentile(gh, 99)),
                            "same_result": bool(torch.equal(ref, s1))}
        except Exception as e:   # report, do not fail the bench line
            lat["graph"] = {"error": str(e)[:200]}
        # closed loop from pinned host memory: frame in -> (shift, f_min) back on the host
        hf1 = frames[:1].cpu().pin_memory()
        hsh = torch.empty((1, 2), dtype=torch.int32).pin_memory()
        hfm = torch.empty((1,), dtype=torch.float64).pin_memory()
        for _ in range(20):
            plan.align_host(hf1, hsh, hfm)
        ws = []
        for _ in range(200):
            t0 = time.perf_counter()
            plan.align_host(hf1, hsh, hfm)
            ws.append((time.perf_counter() - t0) * 1e3)
        lat["frame_to_shift_host"] = {"p50_ms": float(np.percentile(ws, 50)), "p99_ms": float(np.percentile(ws, 99)),
                                      "api": "moco_align_host, 1 pinned frame in, shift + f_min out"}

    # ---- context: the paper's own setting (downsample once, w = min(m,n)/3 of the
    # 256x256 coarse frame = 85), FFT path; the paper quotes ~23 frames/s for its Java
    # implementation on 512x512 videos (hardware not stated)
    paper = None
    if rank == 0 and spec.index == 2 and not args.no_paper:
        pw = 85
        pp = Plan(spec.m, spec.n, pw, 1, spec.dtype, 12, device=local)
        pp.set_template(template)
        nfr = min(Tl, 2048)
        sub = frames[:nfr]
        ps_, pf_, pc_ = shifts[:nfr], fmin[:nfr], corrected[:nfr]
        pp.align_into(sub, ps_, pf_, pc_)
        torch.cuda.synchronize()
        a_ = torch.cuda.Event(enable_timing=True)
        b_ = torch.cuda.Event(enable_timing=True)
        a_.record()
        for _ in range(3):
            pp.align_into(sub, ps_, pf_, pc_)
        b_.record()
        torch.cuda.synchronize()
        paper = {"workload": f"{nfr} frames of 512x512 uint16, levels=1, w={pw} at 256x256 (PAPER.md:49 defaults)",
                 "algo": pp.algo, "value": 3 * nfr / (a_.elapsed_time(b_) / 1e3), "unit": UNIT,
                 "paper_java": "22.7-24.3 frames/s on 512x512 videos, hardware not stated (PAPER.md:56-60)"}
        pp.close()

    # ---- template preparation (S0, once per plan; not in the per-frame time)
    tprep = None
    if rank == 0:
        ts = []
        for _ in range(5):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            plan.set_template(template)   # (synchronises its stream)
            ts.append((time.perf_counter() - t0) * 1e3)
        tprep = {"ms_p50": float(np.percentile(ts, 50)), "api": "moco_set_template + stream sync",
                 "note": "pyramid, g_b, b^2 prefix tables, tensor-core B tiles, template spectrum"}

    # ---- C1 single-frame latency (256x256, w=20, no downsampling)
    lat_c1 = None
    if rank == 0 and spec.index == 2 and not args.no_paper:
        s1spec = config_spec(1, T=8)
        st1 = make_stack(s1spec, 0, 8, device=dev)
        p1 = Plan(256, 256, 20, 0, "u16", 12, device=local)
        p1.set_template(st1.template)
        o1 = st1.frames[:1]
        a1s = torch.empty((1, 2), dtype=torch.int32, device=dev)
        a1f = torch.empty((1,), dtype=torch.float64, device=dev)
        a1c = torch.empty_like(o1)
        for _ in range(20):
            p1.align_into(o1, a1s, a1f, a1c)
        ts = []
        for _ in range(200):
            a_ = torch.cuda.Event(enable_timing=True)
            b_ = torch.cuda.Event(enable_timing=True)
            a_.record()
            p1.align_into(o1, a1s, a1f, a1c)
            b_.record()
            b_.synchronize()
            ts.append(a_.elapsed_time(b_))
        lat_c1 = {"p50_ms": float(np.percentile(ts, 50)), "p99_ms": float(np.percentile(ts, 99)),
                  "workload": "C1 shape: 1 frame of 256x256 u16, w=20, levels=0, corrected written"}
        p1.close()

    # ---- measured ALU peaks (moco_probe_peaks) next to the derived FP32 figure
    alu_peaks = None
    try:
        from paper_1506_06039_b200 import probe_peaks
        alu_peaks = probe_peaks(local)
        alu_peaks["derived_fp32_tflops"] = 148 * 128 * 2 * peaks["sm_max_mhz"] * 1e6 / 1e12
    except Exception as e:
        alu_peaks = {"error": str(e)[:160]}

    # ---- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        # pinned buffers on the GPU's own NUMA node (allocated from its local CPUs; the
        # affinity is restored after the measurement)
        aff0 = os.sched_getaffinity(0)
        local_cpus = gpu_local_cpus(dev)
        if local_cpus:
            os.sched_setaffinity(0, local_cpus)
        hf = frames.cpu().pin_memory()
        hc = torch.empty_like(hf).pin_memory()
        hs = torch.empty((Tl, 2), dtype=torch.int32).pin_memory()
        hfm = torch.empty((Tl,), dtype=torch.float64).pin_memory()
        plan.align_host(hf, hs, hfm, hc)
        # the copy ceiling of these very buffers (host pages of a pinned allocation land on
        # either of the host's memory nodes: the same binary measures ~57 k or ~87 k
        # frames/s from one process to the next, stable within a process)
        ceil = pinned_ceiling(hf, hc, dev)
        if world > 1:
            dist.barrier()
        ksteps = 4
        t0 = time.perf_counter()
        for _ in range(ksteps):
            plan.align_host(hf, hs, hfm, hc)
        dt = torch.tensor([(time.perf_counter() - t0) / ksteps], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        e2e = {"value": world * Tl / float(dt.item()), "unit": UNIT,
               "h2d_bytes_per_step": int(hf.numel() * esz * world),
               "d2h_bytes_per_step": int((hc.numel() * esz + hs.numel() * 4 + hfm.numel() * 8) * world),
               "api": "moco_align_host (pinned host frames in, shifts/f_min/corrected out)",
               "host_cpus": len(local_cpus) if local_cpus else None,
               "pcie_same_buffers": ceil}
        if "ceiling_fps" in ceil:
            e2e["frac_of_pcie_ceiling"] = e2e["value"] / (world * ceil["ceiling_fps"])
        del hf, hc
        os.sched_setaffinity(0, aff0)

    # ---- parity on a bounded sample of the timed workload + the CPU oracle baseline
    # (rank 0, N=1 only): the same oracle run gives both
    cpu = None
    parity = None
    if rank == 0 and world == 1 and not args.no_cpu:
        # the latency and paper-setting runs above reused the output buffers: re-run the
        # (deterministic) step so the buffers hold the timed workload's results
        plan.align_into(frames, shifts, fmin, corrected)
        torch.cuda.synchronize()
        parity = parity_report(frames, template, shifts, fmin, corrected, spec)
        cpu = {"value": parity["oracle_fps"], "unit": UNIT, "cores": parity["cores"], "kind": "oracle",
               "cpu_model": parity["cpu_model"],
               "sample": f"{parity['frames_checked']} frames ({parity['sample']}), oracle fp64 numpy brute "
                         f"force, {parity['cores']}-process pool, {parity['oracle_s']:.1f} s wall"}

    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
               "vs_baseline": None, "dtype": "u16" if spec.dtype == "u16" else "f32", "data": "synthetic",
               "config": dict(workload_config(spec, world, plan.algo),
                              **({"results_gather": gather_mode} if world > 1 else {})),
               "roofline": roofline,
               "step_roofline": {"fps": step_roof, "frac": value / world / step_roof,
                                 "hbm_fps": hbm_roof_fps, "alu_fps": alu_roof_fps,
                                 "hbm_fps_8tbs": 8000e9 / (2 * spec.m * spec.n * esz),
                                 "frac_8tbs": value / world / min(8000e9 / (2 * spec.m * spec.n * esz), alu_roof_fps),
                                 "model": "BASELINE.md §2: slower of (in+out bytes)/HBM and §8(d) FLOPs/FP32"},
               "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches_per_step * args.steps,
               "latency_1frame": lat, "latency_1frame_c1": lat_c1, "template_prep": tprep,
               "parity": parity, "alu_peaks_measured": alu_peaks, "paper_setting": paper, "clocks": clocks}
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
