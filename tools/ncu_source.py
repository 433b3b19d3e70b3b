"""Per-instruction view of an .ncu-rep source page: python tools/ncu_source.py rep [top] [--range lo hi]
Prints opcode histogram weighted by executed count and the top stalled instructions."""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
lines = raw.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
hdr = rows[0]
ia, isrc, isamp, iex = hdr.index("Address"), hdr.index("Source"), hdr.index("# Samples"), hdr.index("Instructions Executed")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
ops = collections.Counter(); tot_ex = 0; tot_s = 0
data = []
for k, r in enumerate(rows[1:]):
    if len(r) <= iex or not r[iex].isdigit():
        continue
    ex, s = int(r[iex]), int(r[isamp] or 0)
    op = r[isrc].split()
    name = op[1] if op and op[0].startswith("@") else (op[0] if op else "?")
    ops[name.split(".")[0]] += ex
    tot_ex += ex; tot_s += s
    data.append((k, r[isrc].strip(), ex, s, {hdr[i]: int(r[i] or 0) for i in stall_cols if (r[i] or "0") != "0"}))
print(f"instructions executed {tot_ex}, samples {tot_s}, static instrs {len(data)}")
for name, c in ops.most_common(18):
    print(f"  {name:10s} {c:12d} {100.0*c/tot_ex:5.1f}%")
agg = collections.Counter()
for d in data:
    for k2, v in d[4].items():
        agg[k2] += v
print("stall totals:", ", ".join(f"{k} {v}" for k, v in agg.most_common(10)))
print("top stalled instructions:")
for d in sorted(data, key=lambda d: -d[3])[:top]:
    print(f"  #{d[0]:5d} ex={d[2]:9d} samp={d[3]:6d} {d[1][:70]:70s} {dict(sorted(d[4].items(), key=lambda kv:-kv[1])[:3])}")
if "--dump" in sys.argv:
    lo, hi = int(sys.argv[sys.argv.index("--dump")+1]), int(sys.argv[sys.argv.index("--dump")+2])
    for d in data[lo:hi]:
        print(f"  #{d[0]:5d} ex={d[2]:8d} s={d[3]:5d} {d[1][:90]}")
if "--byop" in sys.argv:
    byop = collections.Counter(); cnt = collections.Counter()
    for d in data:
        op = d[1].split()
        name = op[1] if op and op[0].startswith("@") else (op[0] if op else "?")
        byop[name.split(".")[0]] += d[3]; cnt[name.split(".")[0]] += d[2]
    print("samples by opcode (where warps sit):")
    for name, c in byop.most_common(16):
        print(f"  {name:10s} samples {c:8d} {100.0*c/tot_s:5.1f}%   executed {cnt[name]:12d}  samples/1k-exec {1000.0*c/max(cnt[name],1):7.2f}")
