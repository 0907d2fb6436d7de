"""Attribute an ncu SASS source page (csv) to CUDA source lines via nvdisasm -g line info.
usage: sass_lines.py <ncu-rep> <kernel regex> <mangled name> <all.sass> [top]"""
import collections, csv, re, subprocess, sys

rep, kre, name, sassf = sys.argv[1:5]
top = int(sys.argv[5]) if len(sys.argv) > 5 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-name",
                      "regex:" + kre], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
data = [r for r in rows[2:] if len(r) == len(h)]
lines = open(sassf).read().split("\n")
start = [i for i, l in enumerate(lines) if l.startswith("//---") and name in l][0]
ins, cur = [], None
for l in lines[start + 1:]:
    if l.startswith("//---------------------"):
        break
    m = re.match(r'\s*//## File "(.*)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip(), cur))
iI, iW, iA = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)"), h.index("Address")


def fl(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


base = int(data[0][iA], 16)
byoff = {o: s for o, _, s in ins}
cnt, smp = collections.Counter(), collections.Counter()
for r in data:
    if not r[iA].startswith("0x"):
        break
    off = int(r[iA], 16) - base
    if off not in byoff:
        break
    cnt[byoff[off]] += fl(r[iI])
    smp[byoff[off]] += fl(r[iW])
tot, ts = sum(cnt.values()), sum(smp.values()) or 1
srcs = {}
print(f"{name}: {tot / 1e6:.2f} M warp instructions")
for s_, v in sorted(cnt.items(), key=lambda x: -x[1])[:top]:
    f, ln = s_ if s_ else ("?", 0)
    if f not in srcs:
        try:
            srcs[f] = open("paper_1506_06039_b200/csrc/" + f).read().split("\n")
        except OSError:
            srcs[f] = []
    txt = srcs[f][ln - 1].strip()[:80] if 0 < ln <= len(srcs[f]) else ""
    print("%5.3f instr %5.3f samp %s:%d  %s" % (v / tot, smp[s_] / ts, f, ln, txt))
