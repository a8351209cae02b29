"""Warp-stall samples of an ncu capture aggregated per CUDA source line.
Usage: ncu_lines.py REP.ncu-rep OBJ.o KERNEL_SUBSTRING [top]
(the object must be the -lineinfo build the capture ran; SASS offsets from the
ncu source page are matched to nvdisasm -g line info)."""
import collections, csv, io, os, re, subprocess, sys, tempfile

rep, obj, pat = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{pat}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hi]
data = [dict(zip(hdr, r)) for r in rows[hi + 1:] if len(r) == len(hdr)]
base = int(data[0]["Address"], 16)
stall_cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    dis = subprocess.run(["nvdisasm", "-g", os.path.join(d, cub)], capture_output=True, text=True).stdout
line_of = {}
cur, fn = None, None
for l in dis.splitlines():
    m = re.search(r"\.text\.(\S+):", l)
    if m:
        fn = m.group(1)
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]+)\*/", l)
    if m and fn and pat in fn:
        line_of[int(m.group(1), 16)] = cur
agg = collections.Counter()
why = collections.defaultdict(collections.Counter)
for r in data:
    off = int(r["Address"], 16) - base
    n = int(r["Warp Stall Sampling (All Samples)"] or 0)
    k = line_of.get(off, ("?", 0))
    agg[k] += n
    for c in stall_cols:
        why[k][c] += int(r[c] or 0)
tot = sum(agg.values())
print(f"total samples {tot}")
for k, v in agg.most_common(top):
    reasons = ", ".join(f"{c[6:]} {n}" for c, n in why[k].most_common(3) if n)
    print(f"{v:6d} {100 * v / tot:5.1f}%  {k[0]}:{k[1]}  ({reasons})")
