"""Per-instruction view of an exported ncu source page (CSV): python tools/src_csv.py file.csv [--dump lo hi] [--regions]
Opcode histogram, stall totals, and the instruction stream with samples (where warps sit)."""
import csv, io, sys, collections
lines = open(sys.argv[1]).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
hdr = rows[0]
isrc, isamp, iex = hdr.index("Source"), hdr.index("# Samples"), hdr.index("Instructions Executed")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
data = []
for k, r in enumerate(rows[1:]):
    if len(r) <= iex or not r[iex].isdigit():
        continue
    data.append((k, r[isrc].strip(), int(r[iex]), int(r[isamp] or 0),
                 {hdr[i][6:]: int(r[i] or 0) for i in stall_cols if (r[i] or "0") != "0"}))
tot_ex = sum(d[2] for d in data); tot_s = sum(d[3] for d in data)
def opname(src):
    op = src.split()
    name = op[1] if op and op[0].startswith("@") else (op[0] if op else "?")
    return name.split(".")[0]
ops = collections.Counter(); samp = collections.Counter()
for d in data:
    ops[opname(d[1])] += d[2]; samp[opname(d[1])] += d[3]
print(f"executed {tot_ex} samples {tot_s} static {len(data)}")
for n, c in ops.most_common(16):
    print(f"  {n:8s} ex {c:11d} {100*c/tot_ex:5.1f}%  samples {samp[n]:8d} {100*samp[n]/tot_s:5.1f}%")
agg = collections.Counter()
for d in data:
    for k2, v in d[4].items():
        agg[k2] += v
print("stalls:", ", ".join(f"{k} {v}" for k, v in agg.most_common(9)))
if "--dump" in sys.argv:
    i = sys.argv.index("--dump"); lo, hi = int(sys.argv[i + 1]), int(sys.argv[i + 2])
    for d in data[lo:hi]:
        st = ",".join(f"{k}:{v}" for k, v in sorted(d[4].items(), key=lambda kv: -kv[1])[:2])
        print(f"#{d[0]:5d} ex={d[2]:9d} s={d[3]:6d} {d[1][:84]:84s} {st}")
if "--regions" in sys.argv:
    # group consecutive instructions with equal executed count: a region = one basic block / loop body
    reg = []
    for d in data:
        if reg and reg[-1][2] == d[2]:
            reg[-1][1] = d[0]; reg[-1][3] += d[3]; reg[-1][4] += 1
        else:
            reg.append([d[0], d[0], d[2], d[3], 1])
    for r in sorted(reg, key=lambda r: -r[3])[:25]:
        print(f"  #{r[0]:5d}-{r[1]:5d} n={r[4]:5d} ex/instr={r[2]:10d} samples={r[3]:8d} {100*r[3]/tot_s:5.1f}%  samples/instr={r[3]/r[4]:8.1f}")
if "--phases" in sys.argv:
    # split the stream at DMMA clusters (gaps < 60 instructions belong to the same cluster)
    idx = [i for i, d in enumerate(data) if opname(d[1]) == "DMMA"]
    clusters = []
    for i in idx:
        if clusters and i - clusters[-1][1] < 60:
            clusters[-1][1] = i
        else:
            clusters.append([i, i])
    pos = 0
    for lo, hi in clusters + [[len(data), len(data)]]:
        seg = data[pos:lo]
        if seg:
            ex = max(d[2] for d in seg)
            print(f"  non-DMMA #{pos:5d}-{lo:5d} instr={len(seg):5d} exmax={ex:9d} samples={sum(d[3] for d in seg):8d} {100*sum(d[3] for d in seg)/tot_s:5.1f}%  dyn-instr={sum(d[2] for d in seg)/max(ex,1):8.1f}")
        seg = data[lo:hi + 1]
        if seg:
            ex = max(d[2] for d in seg)
            nd = sum(1 for d in seg if opname(d[1]) == "DMMA")
            print(f"  DMMA     #{lo:5d}-{hi:5d} instr={len(seg):5d} dmma={nd:4d} samples={sum(d[3] for d in seg):8d} {100*sum(d[3] for d in seg)/tot_s:5.1f}%")
        pos = hi + 1
