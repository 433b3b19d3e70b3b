"""In-order issue model of one SM sub-partition running W copies of a straight-line SASS region.
python tools/sass_sim.py sass.txt START END [W] [OFFSET]
Latencies (B200, measured by tools/probe_fp64.cu / probe_mix.cu): FP64 result 8.4 clk, FP64 pipe busy 2 clk
per warp instruction; ALU-pipe ops (LOP3/IADD3/SHF/SEL/FSEL/ISETP/...) share the FP64 dispatch slot (1 clk)."""
import re, sys
FP64 = ("DFMA", "DMUL", "DADD", "DSETP")
ALU = ("LOP3", "IADD3", "SHF", "SEL", "FSEL", "ISETP", "PLOP3", "CS2R", "MOV", "FMNMX", "LEA", "R2UR", "PRMT", "IABS", "FSETP")
LAT = {"fp64": 8.4, "alu": 4.5, "fma": 4.5, "lds": 30, "ldg": 600, "mufu": 22, "shfl": 25, "other": 5}
def regs64(tok, wide):
    m = re.search(r"R(\d+)", tok)
    if not m or "RZ" in tok and not m: return []
    r = int(m.group(1))
    return [r, r + 1] if wide else [r]
def parse(line):
    m = re.match(r"/\*[0-9a-f]+\*/\s+(@!?U?P\d+\s+)?([A-Z0-9_.]+)\s*(.*?)\s*;", line)
    if not m: return None
    pred, op, args = m.group(1), m.group(2), m.group(3)
    base = op.split(".")[0]
    toks = [t.strip() for t in re.split(r",(?![^\[]*\])", args)] if args else []
    wide = base in FP64 or ".64" in op or base in ("DFMA",)
    kind = "fp64" if base in FP64 else "alu" if base in ALU else "lds" if base == "LDS" else "ldg" if base in ("LDG", "LDL", "LD") else \
           "mufu" if base == "MUFU" else "shfl" if base == "SHFL" else "fma" if base in ("IMAD", "FFMA", "FMUL", "FADD") else "other"
    dst, src = [], []
    preds_dst, preds_src = [], []
    if pred: preds_src.append(re.search(r"P\d+", pred).group(0))
    store = base in ("STS", "STG", "STL", "ST", "BRA", "BAR", "EXIT", "UBLKPF", "BSYNC", "BSSY", "WARPSYNC", "NOP")
    for i, t in enumerate(toks):
        is_dst = (i == 0 and not store)
        if base in ("DSETP", "ISETP", "FSETP", "PLOP3") and i <= 1 and re.fullmatch(r"!?U?P\d+|PT", t):
            if t != "PT": preds_dst.append(t.strip("!"))
            continue
        ps = re.findall(r"(?<![A-Z])P\d+", t)
        if is_dst and re.match(r"\[?R\d+", t) and not t.startswith("["):
            w = wide and base != "DSETP"
            if base == "MUFU": w = False
            if base == "LDS" or base == "LDG": w = ".64" in op; 
            if ".128" in op: dst += [int(re.search(r"R(\d+)", t).group(1)) + k for k in range(4)]
            else: dst += regs64(t, w)
        else:
            for r in re.findall(r"R(\d+)", t):
                r = int(r)
                w = (base in FP64) or (base in ("STS", "STG") and ".64" in op and not t.startswith("["))
                if base == "MUFU": w = False
                src += [r, r + 1] if w else [r]
            preds_src += [p for p in ps]
    return dict(op=op, kind=kind, dst=dst, src=src, pd=preds_dst, ps=preds_src, text=line.strip()[:70])
def simulate(instrs, W, offset):
    n = len(instrs)
    pc = [0] * W
    ready = [dict() for _ in range(W)]   # reg -> time ready
    next_ok = [w * offset for w in range(W)]
    fp_free = 0.0; t = 0.0; done = 0
    stall_at = [0.0] * n
    last = 0
    while done < W:
        issued = False
        order = sorted(range(W), key=lambda w: (w != last, w))  # greedy-then-oldest flavour
        for w in order:
            if pc[w] >= n or next_ok[w] > t: continue
            ins = instrs[pc[w]]
            rt = max([ready[w].get(("R", r), 0) for r in ins["src"]] + [ready[w].get(("P", p), 0) for p in ins["ps"]] + [0])
            if rt > t: continue
            if ins["kind"] in ("fp64", "alu") and fp_free > t: continue
            cost = 2 if ins["kind"] == "fp64" else 1
            if ins["kind"] in ("fp64", "alu"): fp_free = t + cost
            lat = LAT[ins["kind"]]
            for r in ins["dst"]: ready[w][("R", r)] = t + lat
            for p in ins["pd"]: ready[w][("P", p)] = t + lat + 4
            pc[w] += 1; next_ok[w] = t + 1; last = w; issued = True
            if pc[w] >= n: done += 1
            break
        if not issued:
            for w in range(W):
                if pc[w] < n: stall_at[pc[w]] += 1.0 / W
        t += 1
    return t, stall_at
if __name__ == "__main__":
    lines = [l for l in open(sys.argv[1]) if l.startswith("/*")]
    a, b = int(sys.argv[2]), int(sys.argv[3])
    W = int(sys.argv[4]) if len(sys.argv) > 4 else 2
    off = int(sys.argv[5]) if len(sys.argv) > 5 else 0
    ins = [p for p in (parse(l) for l in lines[a:b]) if p]
    nf = sum(1 for i in ins if i["kind"] == "fp64"); na = sum(1 for i in ins if i["kind"] == "alu")
    t, st = simulate(ins, W, off)
    print(f"{len(ins)} instrs, fp64 {nf}, alu {na}: W={W} offset={off}: {t:.0f} clk; fp64 pipe busy {2*nf*W/t:.2%}, fp64+alu slot {(2*nf+na)*W/t:.2%}")
    if "--top" in sys.argv:
        for k in sorted(range(len(ins)), key=lambda k: -st[k])[:25]:
            print(f"  {k+a:5d} stall {st[k]:6.1f}  {ins[k]['text']}")
