"""Aggregate ncu SASS stall samples by CUDA source line: ncu_lines.py REP KERNEL_MANGLED [N]."""
import csv, re, subprocess, sys, os, tempfile
rep, fn = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
lib = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1904_10548_b200/lib/libwmpc.so")
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=tmp, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
sass = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout.split("\n")
start = next(i for i, l in enumerate(sass) if l.startswith(".text." + fn + ":"))
off2line, cur = {}, None
for l in sass[start + 1:]:
    if l.startswith(".text.") and l.rstrip().endswith(":"): break
    m = re.search(r'##\s*File "([^"]+)", line (\d+)', l)
    if m: cur = (m.group(1).split("/")[-1], int(m.group(2))); continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if m and cur: off2line[int(m.group(1), 16)] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", *sys.argv[4:]], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
if rows and rows[0] and rows[0][0] == "Kernel Name":
    rows = rows[1:]
h = rows[0]; data = [r for r in rows[1:] if r and r[0].startswith("0x")]
i_s = h.index(os.environ.get("NCU_COL", "Warp Stall Sampling (All Samples)"))
stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
base = min(int(r[0], 16) for r in data)
agg, reasons = {}, {}
tot = 0.0
for r in data:
    s = float(r[i_s] or 0); tot += s
    key = off2line.get(int(r[0], 16) - base, ("?", 0))
    agg[key] = agg.get(key, 0) + s
    rs = reasons.setdefault(key, {})
    for i in stall_cols:
        v = float(r[i] or 0)
        if v: rs[h[i]] = rs.get(h[i], 0) + v
srcs = {}
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    fnm, ln = k
    if fnm not in srcs:
        p = os.path.join(os.path.dirname(lib), "..", "csrc", fnm)
        srcs[fnm] = open(p).read().split("\n") if os.path.exists(p) else []
    text = srcs[fnm][ln - 1].strip()[:70] if srcs[fnm] and ln else ""
    rs = sorted(reasons[k].items(), key=lambda kv: -kv[1])[:2]
    print(f"{v / tot * 100:5.1f}% {fnm}:{ln:<4d} {text:70s} {[(a.replace('stall_', ''), round(b / max(v, 1) * 100)) for a, b in rs]}")
