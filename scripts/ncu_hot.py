"""Top stall-sampled SASS instructions of an ncu report (source page)."""
import csv, io, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
lines = out.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
data = rows[1:]
tot = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg = {s: 0 for s in stalls}
for r in data:
    for s in stalls:
        try:
            agg[s] += int(r[ix[s]] or 0)
        except ValueError:
            pass
print("total samples", tot)
print({k: round(v / tot, 3) for k, v in sorted(agg.items(), key=lambda kv: -kv[1]) if v / max(tot, 1) > 0.01})
data.sort(key=lambda r: -int(r[ix["Warp Stall Sampling (All Samples)"]] or 0))
for r in data[:top]:
    n = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    top_st = sorted(((int(r[ix[s]] or 0), s) for s in stalls), reverse=True)[:2]
    print(f"{n / tot:6.3f} {r[ix['Address']][-5:]} {r[ix['Source']].strip()[:60]:60s} {top_st}")
