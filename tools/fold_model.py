"""FP64 instruction-count model of the fold kernel: python tools/fold_model.py n"""
import sys
CH = 15  # scalar chain FP64 ops
def model(n, G, P):
    NS = -(-n // G)
    useful = P * n * NS  # per lane, FMA units (P*n^2 / G)
    tot = P + CH  # head
    shfl = 2 * P if G > 1 else 0
    for c in range(n):
        bc, gc = divmod(c, G)
        peel = gc == G - 1
        live = NS - bc - (1 if peel else 0)
        tot += (2 * P + 3) * live
        if c + 1 < NS * G and (bc + (1 if peel else 0)) < NS:
            tot += P + CH
            shfl += (2 * P + 2) if G > 1 else 0
    tri = NS * G * (NS * G + 1) // 2
    ts = tri + ((G - tri % 16) + 16) % 16
    groups = 227 * 1024 // (ts * 8)
    thr = groups * G // 128 * 128
    thr = min(thr, 256)
    regs = 2 * (NS * P + (P if G > 1 else 0) + NS)
    return useful / tot, tot, shfl, thr, regs
n = int(sys.argv[1])
for G in (1, 2, 4, 8, 16):
    for P in (4, 6, 8, 12, 16, 24):
        if -(-n // G) * P > 112: continue
        e, tot, shfl, thr, regs = model(n, G, P)
        if thr < 128: continue
        print(f"n={n} G={G:2d} P={P:2d} NS={-(-n//G):2d}: eff {e:.3f} fp64/lane-step {tot:5d} shfl {shfl:4d} ({shfl/tot:.2f}/fp64) T={thr} regs~{regs}")
