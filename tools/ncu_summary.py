"""Summarise an ncu report (raw page): key counters + top stall reasons + hottest SASS."""
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, u = rows[0], rows[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers", "launch__block_size",
        "launch__grid_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
for v in rows[2:]:
    print("==", v[h.index("Kernel Name")][:80])
    for n in want:
        if n in h:
            print(f"  {n} = {v[h.index(n)]} {u[h.index(n)]}")
    st = []
    for i, n in enumerate(h):
        if n.startswith("smsp__pcsamp_warps_issue_stalled") and not n.endswith("not_issued"):
            try:
                st.append((float(v[i]), n.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(x for x, _ in st) or 1
    print("  stalls:", ", ".join(f"{n} {100*x/tot:.0f}%" for x, n in sorted(st, reverse=True)[:8]))
if len(sys.argv) > 2:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rr = list(csv.reader(src.splitlines()))
    hh = rr[1]
    ia, isrc = hh.index("Address"), hh.index("Source")
    ist, iex = hh.index("Warp Stall Sampling (All Samples)"), hh.index("Instructions Executed")
    data = []
    for r in rr[2:]:
        try:
            data.append((int(r[ist] or 0), int(r[iex] or 0), r[ia][-5:], r[isrc][:80]))
        except (ValueError, IndexError):
            pass
    for d in sorted(data, reverse=True)[: int(sys.argv[2])]:
        print("  ", d)


def pc_reasons(rep, top=15):
    """Per-PC stall reason breakdown for the hottest SASS instructions."""
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rr = list(csv.reader(src.splitlines()))
    hh = rr[1]
    ist = hh.index("Warp Stall Sampling (All Samples)")
    rc = [i for i, n in enumerate(hh) if n.startswith("stall_") and "Not Issued" not in n]
    data = []
    for r in rr[2:]:
        try:
            data.append((int(r[ist] or 0), r))
        except (ValueError, IndexError):
            pass
    for n, r in sorted(data, key=lambda x: -x[0])[:top]:
        rs = sorted(((int(r[i] or 0), hh[i][6:]) for i in rc), reverse=True)[:3]
        print(f"  {n:6d} {r[hh.index('Address')][-5:]} {r[hh.index('Source')][:60]:60s} {rs}")


if len(sys.argv) > 3:
    pc_reasons(rep, int(sys.argv[3]))
