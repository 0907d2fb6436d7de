"""Build profiles/ncu_traffic.json (bench.py's roofline 'traffic') from ncu --set full reports:
DRAM bytes (read + write) per frame of each kernel kind.
usage: ncu_traffic.py <c2_tc.ncu-rep> <frames> [<c3_fft.ncu-rep> <frames>] > profiles/ncu_traffic.json"""
import csv
import json
import subprocess
import sys

KINDS_TC = {"k_tc_prep": "tc_prep", "k_tc_coarse": "coarse", "k_refine_tc": "refine", "k_ga_pieces": "apply",
            "k_refine_pick": "apply"}
KINDS_FFT = {"k_fft2_rows": "tc_prep", "k_fft2_cols": "coarse", "k_fft2_score": "tc_score", "k_fft2_rescore": "tc_score"}


SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}


def rows(rep):
    """Each kernel launch as {metric: value in bytes / microseconds}."""
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(raw.splitlines()))
    h, u = r[0], r[1]
    for v in r[2:]:
        d = {}
        for i, k in enumerate(h):
            try:
                d[k] = float(v[i].replace(",", "")) * SCALE.get(u[i], 1)
            except ValueError:
                d[k] = v[i]
        yield d


def build(rep, frames, kinds, cfg, algo, out):
    agg = {}
    for d in rows(rep):
        name = d["Kernel Name"]
        short = name.replace("void ", "").split("<")[0].split("(")[0]
        kind = kinds.get(short)
        if not kind:
            continue
        e = agg.setdefault(kind, {"kernel": [], "bytes": 0.0, "dur": 0.0})
        e["kernel"].append(name.split("(")[0].replace("void ", ""))
        e["bytes"] += d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
        e["dur"] += d["gpu__time_duration.sum"]
    out.setdefault(cfg, {})[algo] = {
        k: {"kernel": " + ".join(v["kernel"]), "bytes_per_frame": v["bytes"] / frames, "frames_in_capture": frames,
            "duration_us": v["dur"]} for k, v in agg.items()}


out = {}
args = sys.argv[1:]
build(args[0], float(args[1]), KINDS_TC, "C2", "tc", out)
if len(args) > 3:
    build(args[2], float(args[3]), KINDS_FFT, "C3", "fft", out)
out["_source"] = ("ncu --set full --clock-control none captures (tools/profile_all.sh): C2 tensor-core path, "
                  "MOCO_BATCH_WAVES=1 tools/profile_run.py --frames 4736 (one 1,184-frame batch, cold cache); C3 FFT "
                  "path, tools/profile_run.py --algo fft, one steady-state sub-batch with --cache-control none "
                  "(warm L2); dram__bytes_read.sum + dram__bytes_write.sum per launch / frames per launch, bytes; "
                  "duration_us = gpu__time_duration.sum of the capture's launches")
print(json.dumps(out, indent=1))
