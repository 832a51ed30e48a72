"""Attribute ncu SASS-level stall samples to CUDA source lines.

    python scripts/ncu_lines.py REPORT MANGLED_KERNEL_NAME [top]

Aligns the report's SASS listing (address order) with nvdisasm --print-line-info
of the in-tree library (same build that was profiled) by instruction offset.
"""
import collections, csv, io, re, subprocess, sys, tempfile, os, glob

rep, fn = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
lib = os.path.join(os.path.dirname(__file__), "..", "paper_2410_01657_b200", "lib", "libhgnn_b200.so")
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
lines_by_off = {}
for cub in glob.glob(os.path.join(tmp, "*.cubin")):
    full = subprocess.run(["nvdisasm", "--print-line-info", cub], capture_output=True, text=True).stdout
    start = full.find(f"\n.text.{fn}:")
    if start < 0:
        continue
    end = full.find("//---------------------", start)
    txt = full[start:end if end > 0 else len(full)]
    cur = None
    for line in txt.splitlines():
        m = re.search(r'//## File "([^"]+)", line (\d+)', line)
        if m:
            cur = f"{os.path.basename(m.group(1))}:{m.group(2)}"
            continue
        m = re.match(r'\s*/\*([0-9a-f]{4,})\*/\s+(.*)', line)
        if m:
            lines_by_off[int(m.group(1), 16)] = (cur, m.group(2).strip()[:50])
    break
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO("\n".join(out.splitlines()[1:]))))
hdr, data = rows[0], rows[1:]
ix = {h: i for i, h in enumerate(hdr)}
base = int(data[0][ix["Address"]], 16)
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
per_line = collections.defaultdict(collections.Counter)
tot = 0
for r in data:
    n = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    tot += n
    off = int(r[ix["Address"]], 16) - base
    ln = lines_by_off.get(off, ("?", ""))[0]
    for s in stalls:
        v = int(r[ix[s]] or 0)
        if v:
            per_line[ln][s[6:]] += v
print("samples", tot, "mapped offsets", len(lines_by_off))
ranked = sorted(per_line.items(), key=lambda kv: -sum(kv[1].values()))
for ln, c in ranked[:top]:
    s = sum(c.values())
    print(f"{s / tot:6.3f} {ln:28s} {dict(c.most_common(3))}")
if len(sys.argv) > 4:
    print("--- top instructions")
    inst = []
    for r in data:
        n = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        off = int(r[ix["Address"]], 16) - base
        ln, txt = lines_by_off.get(off, ("?", ""))
        inst.append((n, off, ln, r[ix["Source"]].strip()[:70]))
    inst.sort(reverse=True)
    for n, off, ln, txt in inst[:int(sys.argv[4])]:
        print(f"{n / tot:6.3f} {off:6x} {ln:24s} {txt}")
