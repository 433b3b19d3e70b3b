"""Builds profiles/README.md and copies the round's evidence from gpurun_out/ into profiles/.
python tools/make_profile_readme.py [tag]"""
import csv
import json
import re
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
G, P = ROOT / "gpurun_out", ROOT / "profiles"
tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
P.mkdir(exist_ok=True)


def jline(path):
    for line in open(path):
        line = line.strip()
        if line.startswith("{"):
            return json.loads(line)
    return None


out = [f"# Round evidence ({tag}) - one B200, sm_100a\n",
       "Everything here was produced by `tools/round_profile.sh` under `gpurun` (one command, one box): "
       "`bench.py` for both arms, the ncu launch list of the same bench command, one `ncu --set full` capture per "
       "streaming kernel family (kept as raw-metric CSVs: the `.ncu-rep` files together exceed what gpurun returns), "
       "the `nvidia-smi` clock log during the bench, and the BASELINE configurations C1/C3/C4/C5 (`tools/run_configs.py`). "
       "Numbers under ncu are cold-cache and serialised: compare shares, not absolutes.\n"]

bench = jline(G / f"{tag}_bench.json")
ref = jline(G / f"{tag}_bench_reference.json")
if bench:
    shutil.copy(G / f"{tag}_bench.json", P / f"{tag}_bench.json")
    r = bench["roofline"]
    out.append("## Headline (bench.py, N = 1)\n")
    out.append(f"* workload: {bench['config']['workload']}; plan {bench['config']['plan']}")
    hbm_peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (ROOT / "MEASURED_PEAKS.json").exists() else 6540.0
    out.append(f"* **value {bench['value']:.0f} GB/s** ({bench['ms_per_step']:.3f} ms per step, {bench['gpu_launches']} launches in the timed region) - "
               f"the SUSTAINED figure: K steps after 300 ms of untimed back-to-back steps, board on its power cap; "
               f"{100*bench['value']/8000:.1f} % of the nominal 8 TB/s roofline, {100*bench['value']/hbm_peak:.1f} % of the measured copy bandwidth ({hbm_peak:.0f} GB/s); "
               f"clocks {bench['clocks']}")
    if "burst" in bench:
        s = bench["burst"]
        out.append(f"* burst (the same K steps on a settled board): {s['value']:.0f} GB/s = {100*s['value']/8000:.1f} % of 8 TB/s, clocks {s['clocks']}")
    out.append(f"* roofline (stage-1 kernel alone, in situ, settled board): bound {r['bound']}, achieved {r['achieved']:.1f} {r['unit']} = {r['frac']:.3f} of {r['peak']} ({r['peak_source']}); "
               f"DRAM traffic per launch {r['traffic']} B vs algorithmic {r['algorithmic_bytes_per_launch']:.0f} B")
    if "e2e" in bench:
        e = bench["e2e"]
        out.append(f"* e2e through the host-pointer ABI: {e['value']:.1f} GB/s ({e['ms_per_step']:.1f} ms per step, H2D {e['h2d_bytes_per_step']} B per step inside the timed region: PCIe-bound)")
    if "cpu_baseline" in bench:
        c = bench["cpu_baseline"]
        out.append(f"* CPU reference beside it: {c.get('value', 0):.2f} GB/s on {c.get('cores')} host threads ({c.get('kernel_table')}), "
                   f"{c.get('value_without_validation_scan', 0):.1f} GB/s without its serial validation scan; sample: {c.get('sample')}")
    if "parity" in bench:
        out.append(f"* parity of the headline run against the reference on that sample: {bench['parity']}")
    if ref:
        out.append(f"* `bench.py --impl reference`: {ref['value']:.2f} GB/s ({ref['cpu_baseline']['sample']}); same_config = {ref['config'].get('same_config')}")
    c4 = jline(G / f"{tag}_bench_c4.json") if (G / f"{tag}_bench_c4.json").exists() else None
    if c4:
        shutil.copy(G / f"{tag}_bench_c4.json", P / f"{tag}_bench_c4.json")
        out.append(f"* `bench.py --config c4` (BASELINE configs[3], {c4['config']['m_total']} x 16 [A b], {c4['n_gpus']} GPU): {c4['value']:.0f} GB/s, "
                   f"{c4['ms_per_step']:.2f} ms per solve, {c4['gpu_launches']} launches per {c4['steps']} steps; solution {c4['solution']}")
    if ref:
        shutil.copy(G / f"{tag}_bench_reference.json", P / f"{tag}_bench_reference.json")
    if "sweep" in bench:
        out.append("\n## Column sweep at m = 2^27 (BASELINE configs[1]); ms / effective GB/s (8mn / t) / % of 8 TB/s\n")
        if "model_hardware" in bench:
            out.append(f"Roofline model of the reference (perf_model.hpp, `paper_2603_20889_b200/perf_model.py`) with {bench['model_hardware']}; "
                       "`x model` = measured time / model time.\n")
        if "sweep_protocol" in bench:
            out.append(f"Protocol: {bench['sweep_protocol']}; `sustained` = the same reps after 300 ms of back-to-back steps.\n")
        out.append("| n | GiB | TSQR | CholQR2 | SVQB2 | TSQR TFLOP/s (2mn^2) | TSQR sustained GB/s | binding roofline (TSQR): fraction |")
        out.append("|---|---|---|---|---|---|---|---|")
        for row in bench["sweep"]:
            cells = []
            for meth in ("tsqr", "cholqr2", "svqb2"):
                v = row.get(meth, {})
                cells.append((f"{v['ms']:.2f} ms / {v['gbs']:.0f} / {100*v['frac_8TBs']:.1f} %"
                              + (f" / {v['model_ratio']:.2f}x model" if "model_ratio" in v else "")) if "ms" in v else str(v))
            tq = row.get("tsqr", {})
            out.append(f"| {row['n']} | {row['gib']:.0f} | {cells[0]} | {cells[1]} | {cells[2]} | {tq.get('fp64_tflops_2mn2', 0):.1f} | "
                       f"{tq.get('sustained_gbs', 0):.0f} | {tq.get('bound', '')}: {tq.get('frac_of_binding_roofline', 0):.2f} |")

# launch list
lf = G / f"{tag}_launches.csv"
if lf.exists():
    shutil.copy(lf, P / f"{tag}_launches.csv")
    rows = [r for r in csv.reader(l for l in open(lf) if not l.startswith("==")) if len(r) > 5]
    hdr = rows[0]
    if "Kernel Name" in hdr:
        kn, mv = hdr.index("Kernel Name"), hdr.index("Metric Value")
        agg = {}
        for r in rows[1:]:
            try:
                t = float(r[mv].replace(",", ""))
            except ValueError:
                continue
            name = r[kn].split("(")[0].replace("void ", "").replace("sqb::", "").replace("<unnamed>::", "")
            a = agg.setdefault(name, [0, 0.0])
            a[0] += 1
            a[1] += t
        tot = sum(v[1] for v in agg.values())
        out.append(f"\n## Launch list of `bench.py --steps 2 --warmup 1` under ncu ({tag}_launches.csv), share of device time\n")
        out.append("| kernel | launches | total | share |")
        out.append("|---|---|---|---|")
        for name, (cnt, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:16]:
            out.append(f"| `{name}` | {cnt} | {t/1e6:.2f} ms | {100*t/tot:.1f} % |")

# ncu summaries
raws = sorted(G.glob(f"{tag}_*.raw.csv"))
if raws:
    txt = subprocess.run([sys.executable, str(ROOT / "tools" / "ncu_summary_csv.py")] + [str(r) for r in raws],
                         capture_output=True, text=True).stdout
    (P / f"{tag}_ncu_summary.txt").write_text(txt)
    for r in raws:
        shutil.copy(r, P / r.name)
    for r in G.glob(f"{tag}_*.source.csv"):
        shutil.copy(r, P / r.name)
    out.append(f"\n## ncu --set full, one capture per kernel family ({tag}_ncu_summary.txt, raw CSVs beside it)\n")
    out.append("```")
    out.append(txt.replace(str(G) + "/", ""))
    out.append("```")
    # traffic.json for bench.py
    traffic = {}
    for r in raws:
        rows = list(csv.reader(open(r)))
        if len(rows) < 3:
            continue
        hdr = rows[0]
        try:
            rd = float(rows[2][hdr.index("dram__bytes_read.sum")])
            wr = float(rows[2][hdr.index("dram__bytes_write.sum")])
            ur, uw = rows[1][hdr.index("dram__bytes_read.sum")], rows[1][hdr.index("dram__bytes_write.sum")]
        except (ValueError, IndexError):
            continue
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        traffic[r.name.replace(f"{tag}_", "").replace(".raw.csv", "")] = rd * mult.get(ur, 1) + wr * mult.get(uw, 1)
    import math
    kern = {}
    for k, b in traffic.items():
        mnum = re.search(r"_n(\d+)$", k)
        if not mnum or b <= 0:
            continue
        nn = int(mnum.group(1))
        kern[k] = {"bytes": b, "m": 2 ** round(math.log2(b / (8.0 * nn)))}
    tj = {"_source": f"profiles/{tag}_*.raw.csv (ncu --set full): dram__bytes_read.sum + dram__bytes_write.sum per launch of the "
                     "streaming kernel, with the row count of the capture; bench.py scales to its own m", "kernels": kern}
    for nn, key in ((2, "tsqr_thread_n2"), (4, "tsqr_fold_n4"), (8, "tsqr_fold_n8"), (12, "tsqr_fold_n12"), (16, "tsqr_fold_n16"), (24, "tsqr_fold_n24"),
                    (32, "tsqr_mma_n32"), (64, "tsqr_mma_n64")):
        if key in kern:
            tj[f"tsqr_n{nn}"] = kern[key]
    for nn, key in ((8, "gram_thread_n8"), (10, "gram_thread_n10"), (16, "gram_mma_n16"), (32, "gram_mma_n32"), (33, "gram_mma_n33"),
                    (64, "gram_mma_n64")):
        if key in kern:
            tj[f"cholqr2_n{nn}"] = kern[key]
            tj[f"svqb2_n{nn}"] = kern[key]
    (P / "traffic.json").write_text(json.dumps(tj, indent=1))

cf = G / f"configs_{tag}.json"
if cf.exists():
    shutil.copy(cf, P / f"{tag}_configs.json")
    c = json.loads(cf.read_text())
    out.append(f"\n## BASELINE configurations ({tag}_configs.json)\n")
    if "C1" in c:
        out.append("**C1** 1 000 000 x 8 Gaussian, GPU resident / host API / CPU reference (ms), error against the reference's R (bound 64 n eps |X|):\n")
        for meth in ("tsqr", "cholqr2"):
            v = c["C1"][meth]
            out.append(f"* {meth}: {v['gpu_ms_resident']:.3f} / {v['gpu_ms_host_api']:.2f} / {v['cpu_reference_ms']:.1f} ms; err {v['err_vs_reference_tsqr']:.2e} (bound {v['bound']:.2e})")
        v = c["C1"]["svqb2"]
        out.append(f"* svqb2: {v['gpu_ms_resident']:.3f} ms resident, CPU {v['cpu_reference_ms']:.1f} ms, rank {v['rank']}, sigma rel err {v['sigma_rel_err']:.1e}")
    if "C3" in c:
        out.append("\n**C3** 4e7 x 32, controlled condition number (device-side restatement of the reference generator):\n")
        out.append("| kappa | TSQR ms | TSQR |R-R_ref| (bound) | TSQR orth loss | CholQR2 | SVQB2 | CPU ref cholqr2 |")
        out.append("|---|---|---|---|---|---|---|")
        for r in c["C3"]:
            ch = f"{r['cholqr2_ms']:.2f} ms, err vs TSQR {r['cholqr2_err_vs_tsqr']:.1e}, orth {r['cholqr2_orth_loss_2norm']:.1e}" if "cholqr2_ms" in r else r.get("cholqr2")
            sv = f"{r['svqb2_ms']:.2f} ms, rank {r['svqb2_rank']}" if "svqb2_ms" in r else r.get("svqb2")
            out.append(f"| {r['kappa']:.0e} | {r['tsqr_ms']:.2f} | {r['tsqr_err_vs_reference']:.1e} ({r['bound_64_n_eps_normX']:.1e}) | {r['tsqr_orth_loss_2norm']:.1e} | {ch} | {sv} | {r['cpu_reference_cholqr2']} (ref svqb2 rank {r['cpu_reference_svqb2_rank']}) |")
    if "C4" in c:
        v = c["C4"]
        out.append(f"\n**C4** least squares, {v['m']} x {v['n_A']} + rhs on one GPU ({v['bytes']/1e9:.0f} GB streamed once): "
                   + "; ".join(f"{m_}: {v[m_]['ms']:.1f} ms = {v[m_]['gbs']:.0f} GB/s, max |x - planted| {v[m_]['max_abs_err_vs_planted']:.1e}" for m_ in ("tsqr", "cholqr2"))
                   + f"; parity vs CPU reference at 1e7 rows {v['parity_vs_cpu_reference_at_1e7_rows']:.1e}")
    if "C5" in c:
        out.append("\n**C5** Gram matrix at m = 2^24 on the FP64 tensor cores (executed DMMA flops count whole 8x8 tiles of the upper triangle):\n")
        out.append("| n | tsmttsm ms | GB/s | nominal TFLOP/s (2mn^2) | executed DMMA TFLOP/s | DMMA pipe use vs 37.1 | parity err (bound) | TSQR beside it |")
        out.append("|---|---|---|---|---|---|---|---|")
        for r in c["C5"]:
            ts = f"{r['tsqr_ms']:.1f} ms = {r['tsqr_tflops_2mn2']:.1f} TFLOP/s" if "tsqr_ms" in r else "reference rejects n > 64"
            out.append(f"| {r['n']} | {r['tsmttsm_ms']:.2f} | {r['gbs']:.0f} | {r['nominal_tflops_2mn2']:.1f} | {r['executed_dmma_tflops']:.1f} | {100*r['dmma_pipe_util_vs_37.1']:.0f} % | {r['parity_err_F_at_2^17_rows']:.1e} ({r['parity_bound_5_n_eps_normX2']:.1e}) | {ts} |")
        if any("cholqr2_ms" in r for r in c["C5"]):
            out.append("\nCholQR2 (n <= 256) / SVQB2 (n <= 128) at the same sizes (fused solve / multiply + Gram sweeps on the tensor cores; 256 columns: Q = X R^-1 per row slab + the wide SYRK; effective GB/s = 8mn / t):\n")
            out.append("| n | CholQR2 ms | GB/s | R parity err at 2^17 rows (bound 64 n eps |X|) | SVQB2 ms | GB/s |")
            out.append("|---|---|---|---|---|---|")
            for r in c["C5"]:
                if "cholqr2_ms" in r:
                    sv = f"{r['svqb2_ms']:.2f} | {r['svqb2_gbs_effective']:.0f}" if "svqb2_ms" in r else "eigh_small stops at 128 columns | -"
                    out.append(f"| {r['n']} | {r['cholqr2_ms']:.2f} | {r['cholqr2_gbs_effective']:.0f} | {r['cholqr2_parity_err_F_at_2^17_rows']:.1e} ({r['cholqr2_parity_bound_64_n_eps_normX']:.1e}) | {sv} |")

wide = G / f"{tag}_wide.txt"
if wide.exists():
    shutil.copy(wide, P / f"{tag}_wide.txt")
    out.append(f"\n## Wide column counts at m = 2^24 ({tag}_wide.txt; `tools/time_gram_wide.py`)\n\n```\n{wide.read_text().strip()}\n```")

small = G / f"{tag}_small.txt"
if small.exists():
    shutil.copy(small, P / f"{tag}_small.txt")
    out.append(f"\n## The n x n solves alone, one CTA each ({tag}_small.txt; `tools/time_small.py`, Gram matrix of a 65 536-row Gaussian)\n\n```\n{small.read_text().strip()}\n```")
eg = G / f"{tag}_eigh_n128.source_summary.txt"
if eg.exists():
    shutil.copy(eg, P / f"{tag}_eigh_n128.source_summary.txt")
    raw = G / f"{tag}_eigh_n128.raw.csv"
    if raw.exists():
        shutil.copy(raw, P / f"{tag}_eigh_n128.raw.csv")
    head = "\n".join(eg.read_text().splitlines()[:24])
    out.append(f"\n## `eigh_kernel` at 128 x 128 (grouped Jacobi; ncu source page summary, {tag}_eigh_n128.*)\n\n```\n{head}\n```")

clk = G / f"{tag}_clocks.csv"
if clk.exists():
    shutil.copy(clk, P / f"{tag}_clocks.csv")
    rows = list(csv.reader(open(clk)))[1:]
    sm = sorted(int(r[1].split()[0]) for r in rows if len(r) > 3 and r[1].split()[0].isdigit())
    reasons = sorted({r[4].strip() for r in rows if len(r) > 4})
    if sm:
        out.append(f"\n## Clocks during the bench ({tag}_clocks.csv)\n\nSM clock min/median/max {sm[0]}/{sm[len(sm)//2]}/{sm[-1]} MHz over {len(sm)} samples; active reasons seen: {reasons}")
tests = G / f"{tag}_gpu_tests.txt"
if tests.exists():
    out.append(f"\n## GPU tests on the same box\n\n```\n{tests.read_text().strip()}\n```")
alln = G / f"{tag}_all_n.txt"
if alln.exists():
    import re
    shutil.copy(alln, P / f"{tag}_all_n.txt")
    tab = {}
    for l in open(alln):
        mm = re.match(r"(\w+) n=\s*(\d+) m=\s*(\d+)\s+([\d.]+) ms\s+([\d.]+) GB/s", l)
        if mm:
            tab.setdefault(int(mm.group(2)), {})[mm.group(1)] = float(mm.group(5))
    out.append(f"\n## Every column count 1..64 at 16 GiB of X ({tag}_all_n.txt; `tools/time_methods.py`), effective GB/s\n")
    out.append("| n | TSQR | CholQR2 | SVQB2 | tsmttsm |")
    out.append("|---|---|---|---|---|")
    for nn in sorted(tab):
        r = tab[nn]
        out.append(f"| {nn} | {r.get('tsqr', 0):.0f} | {r.get('cholqr2', 0):.0f} | {r.get('svqb2', 0):.0f} | {r.get('tsmttsm', 0):.0f} |")
san = G / f"{tag}_sanitizer.txt"
kept = P / f"{tag}_sanitizer.txt"  # the pool's compute-sanitizer was closed late in round 2: keep the last real pass
if san.exists() and "is closed on this pool" in san.read_text() and kept.exists():
    san = kept
if san.exists():
    out.append(f"\n## compute-sanitizer (memcheck on the GPU parity suite, racecheck on the Gram / TSQR parity tests)\n\n```\n{san.read_text().strip()}\n```")
rw = G / f"{tag}_race_wide.txt"
if rw.exists():
    out.append(f"\nRe-run on the final fused-kernel geometry (32-row solve panels, 2-stage ring):\n\n```\n{rw.read_text().strip()}\n```")
rem = P / "probes" / f"{tag}_remainder_ab.txt"
if rem.exists():
    out.append(f"\n## Remainder-column variants against the padded kernels (profiles/probes/{rem.name})\n\n```\n{rem.read_text().strip()}\n```")
probe = P / "probes" / f"{tag}_tsqr_experiments.txt"
if probe.exists():
    out.append(f"\n## Kernel experiments of this round that were measured and dropped (profiles/probes/{probe.name})\n\n```\n{probe.read_text().strip()}\n```")
(P / "README.md").write_text("\n".join(out) + "\n")
print("wrote", P / "README.md")
