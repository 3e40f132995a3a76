"""Summarise a tools/profile_round.sh output directory into profiles/.

    python tools/summarize_profile.py gpurun_out/r1d r1d

Writes profiles/<tag>_summary.md (bench line, per-kernel launch times from the
recipe's ncu launch list, warm-cache DRAM bytes per kernel, key ncu --set full
metrics of the column and row kernels), copies the launch lists and bench
lines, and updates profiles/traffic.json with the measured DRAM bytes per
application (one profiled step = one forward + one transpose).
"""
import collections
import csv
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")
sys.path.insert(0, ROOT)
from bench import csrc_digest  # noqa: E402  (ties the figures to the kernel sources profiled)


def per_kernel(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: collections.defaultdict(float))
    ids = collections.defaultdict(set)
    for d in data:
        nm = d["Kernel Name"].split("(")[0].replace("void ", "")
        nm = nm.split("<")[0] + "<" + nm.split("<")[1].split(",")[0] + ">" if "<" in nm else nm
        agg[nm][d["Metric Name"]] += float(d["Metric Value"].replace(",", ""))
        ids[nm].add(d["ID"])
    return agg, ids


def last_json(path):
    try:
        return json.loads(open(path).read().strip().splitlines()[-1])
    except Exception:
        return None


FULL_KEYS = [
    ("gpu__time_duration.sum", "duration (ms)"),
    ("l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed", "L1 LSU data-pipe wavefronts % of peak"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe % (fp64 kernels)"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
]


def full_metrics(path):
    rows = list(csv.reader(open(path)))
    if len(rows) < 3:
        return []
    hdr = rows[0]
    out = []
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")[:60]
        vals = {}
        for key, label in FULL_KEYS:
            if key in hdr:
                vals[label] = r[hdr.index(key)]
        out.append((name, vals))
    return out


def fp64_floor(path):
    """FP64 thread instructions (DADD + DMUL + DFMA, predicated on) per captured
    kernel and the time they take on the FP64 pipe at its peak issue rate
    (ncu's own peak: sm__sass_thread_inst_executed_op_dfma_pred_on.sum.peak_sustained
    per cycle, 148 SMs x 64 lanes on B200), at the measured SM clock."""
    rows = list(csv.reader(open(path)))
    if len(rows) < 3:
        return []
    hdr = rows[0]

    def val(r, k):
        return float(r[hdr.index(k)].replace(",", "")) if k in hdr and r[hdr.index(k)] not in ("", "n/a") else None

    out = []
    for r in rows[2:]:
        per = [val(r, f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum.per_cycle_elapsed")
               for op in ("dadd", "dmul", "dfma")]
        cyc = val(r, "smsp__cycles_elapsed.avg")
        peak = val(r, "sm__sass_thread_inst_executed_op_dfma_pred_on.sum.peak_sustained")
        dur = val(r, "gpu__time_duration.sum")
        if None in per or not cyc or not peak or not dur:
            continue
        inst = sum(per) * cyc
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").split("<")[0]
        out.append({"kernel": name, "grid": r[hdr.index("Grid Size")], "duration_ms": dur, "fp64_thread_inst": inst,
                    "dadd": per[0] * cyc, "dmul": per[1] * cyc, "dfma": per[2] * cyc,
                    "floor_ms": inst / peak / (cyc / dur), "peak_per_cycle": peak})
    return out


def main(src, tag):
    os.makedirs(PROF, exist_ok=True)
    lines = [f"# Profile summary `{tag}` (tools/profile_round.sh; B200, clocks not locked)", ""]
    bench = last_json(os.path.join(src, "bench.json"))
    ref = last_json(os.path.join(src, "bench_ref.json"))
    if bench:
        shutil.copy(os.path.join(src, "bench.json"), os.path.join(PROF, f"{tag}_bench.json"))
        lines += ["## bench.py (default: C4 fp64, 20 steps)", "",
                  f"* value {bench['value']:.4g} voxels/s, {bench['ms_per_step']:.3f} ms/step, "
                  f"roofline frac {bench['roofline']['frac']:.3f} of {bench['roofline']['peak']} GB/s, "
                  f"clocks {bench.get('clocks')}",
                  f"* fp32 variant: {bench.get('variants', {}).get('f32')}",
                  f"* e2e: {bench.get('e2e')}", f"* cpu_baseline: {bench.get('cpu_baseline')}", ""]
    if ref:
        shutil.copy(os.path.join(src, "bench_ref.json"), os.path.join(PROF, f"{tag}_bench_ref.json"))
        lines += [f"* reference arm: {ref['value']:.4g} voxels/s ({ref['cpu_baseline']['sample']})", ""]
    traffic = {}
    tpath = os.path.join(PROF, "traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath))
    for dt in ("f64", "f32"):
        lpath = os.path.join(src, f"launches_{dt}.csv")
        tpath_csv = os.path.join(src, f"traffic_{dt}.csv")
        if os.path.exists(lpath):
            shutil.copy(lpath, os.path.join(PROF, f"{tag}_launches_{dt}.csv"))
            agg, ids = per_kernel(lpath)
            tot = sum(m["gpu__time_duration.sum"] for m in agg.values())
            lines += [f"## Launch list, one C4 {dt} step (ncu --metrics gpu__time_duration.sum --clock-control none)", "",
                      "| kernel | launches | mean us | share |", "|---|---|---|---|"]
            for nm, m in sorted(agg.items(), key=lambda kv: -kv[1]["gpu__time_duration.sum"]):
                n = len(ids[nm])
                lines.append(f"| {nm} | {n} | {m['gpu__time_duration.sum'] / n / 1e3:.1f} | "
                             f"{m['gpu__time_duration.sum'] / tot:.3f} |")
            lines.append(f"| total | | {tot / 1e3:.1f} | 1 |")
            lines.append("")
        if os.path.exists(tpath_csv):
            agg, ids = per_kernel(tpath_csv)
            dram = 0.0
            lines += [f"## DRAM bytes, one C4 {dt} step (warm caches: --cache-control none)", "",
                      "| kernel | launches | mean us | DRAM read MB | DRAM write MB | L2 MB |", "|---|---|---|---|---|---|"]
            for nm, m in sorted(agg.items(), key=lambda kv: -kv[1]["gpu__time_duration.sum"]):
                n = len(ids[nm])
                rd, wr = m.get("dram__bytes_read.sum", 0.0), m.get("dram__bytes_write.sum", 0.0)
                dram += rd + wr
                lines.append(f"| {nm} | {n} | {m['gpu__time_duration.sum'] / n / 1e3:.1f} | {rd / 1e6:.1f} | "
                             f"{wr / 1e6:.1f} | {m.get('lts__t_bytes.sum', 0.0) / 1e6:.1f} |")
            per_apply = dram / 2
            traffic[f"C4_{dt}"] = {"bytes_per_apply": per_apply, "profile": tag, "csrc_sha": csrc_digest(),
                                   "how": "ncu dram__bytes_read.sum + dram__bytes_write.sum over one step's "
                                          "launches (--cache-control none), / 2 applications"}
            lines += ["", f"DRAM bytes per application (step / 2): {per_apply / 1e9:.3f} GB", ""]
    fpath = os.path.join(src, "full_f64_raw.csv")
    if os.path.exists(fpath):
        lines += ["## ncu --set full (fp64 kernels of one step, --cache-control none)", ""]
        for name, vals in full_metrics(fpath):
            lines.append(f"* `{name}`: " + ", ".join(f"{k} {v}" for k, v in vals.items()))
        lines.append("")
        fl = fp64_floor(fpath)
        if fl:
            lines += ["## FP64 instruction floor (same capture: one C4 fp64 step)", "",
                      "FP64 thread instructions per kernel (DADD + DMUL + DFMA, predicated on) and the time they "
                      "occupy the FP64 pipe at ncu's peak issue rate (%d thread instructions per cycle = 148 SMs x 64 "
                      "lanes) at the capture's SM clock." % int(fl[0]["peak_per_cycle"]), "",
                      "| kernel | grid | ms | FP64 thread inst (G) | DADD / DMUL / DFMA (G) | floor ms | pipe busy |",
                      "|---|---|---|---|---|---|---|"]
            for k in fl:
                lines.append(f"| {k['kernel']} | {k['grid']} | {k['duration_ms']:.3f} | {k['fp64_thread_inst'] / 1e9:.2f} | "
                             f"{k['dadd'] / 1e9:.2f} / {k['dmul'] / 1e9:.2f} / {k['dfma'] / 1e9:.2f} | "
                             f"{k['floor_ms']:.3f} | {k['floor_ms'] / k['duration_ms']:.2f} |")
            tot_i = sum(k["fp64_thread_inst"] for k in fl)
            tot_f = sum(k["floor_ms"] for k in fl)
            tot_d = sum(k["duration_ms"] for k in fl)
            lines += [f"| step | | {tot_d:.3f} | {tot_i / 1e9:.2f} | | {tot_f:.3f} | {tot_f / tot_d:.2f} |", "",
                      f"One step issues {tot_i / 1e9:.1f} G FP64 thread instructions: {tot_f:.2f} ms of the FP64 pipe at "
                      "100% -- beside the HBM floor of the algorithmic bytes (2 x 5.124 GB / 6.55 TB/s = 1.56 ms) "
                      "the step has a second, slightly higher floor.", ""]
            traffic["C4_f64_fp64_pipe"] = {"fp64_thread_inst_per_step": tot_i, "floor_ms_per_step": tot_f,
                                           "peak_thread_inst_per_cycle": fl[0]["peak_per_cycle"], "profile": tag,
                                           "csrc_sha": csrc_digest(),
                                           "how": "ncu --set full: (dadd + dmul + dfma thread instructions per cycle) x "
                                                  "cycles of every kernel of one step / peak issue rate"}
    f32path = os.path.join(src, "full_f32_raw.csv")
    if os.path.exists(f32path):
        lines += ["## ncu --set full (fp32 row kernels of one C4 step)", ""]
        for name, vals in full_metrics(f32path):
            lines.append(f"* `{name}`: " + ", ".join(f"{k} {v}" for k, v in vals.items()))
        lines.append("")
    cpath = os.path.join(src, "full_c5_raw.csv")
    if os.path.exists(cpath):
        lines += ["## ncu --set full (C5 CGLS fp32: column kernels of one loop)", ""]
        fr = []
        for name, vals in full_metrics(cpath):
            lines.append(f"* `{name}`: " + ", ".join(f"{k} {v}" for k, v in vals.items()))
            if "k_col" in name and "FMA pipe %" in vals:
                fr.append(float(vals["FMA pipe %"].replace(",", "")) / 100.0)
        if fr:
            traffic["C5_cgls_f32"] = {"fp32_pipe_frac": sum(fr) / len(fr), "profile": tag, "csrc_sha": csrc_digest(),
                                      "how": "mean sm__pipe_fma_cycles_active of the captured column kernels"}
        lines.append("")
    traffic = {k: v for k, v in traffic.items() if isinstance(v, dict)}
    json.dump(traffic, open(os.path.join(PROF, "traffic.json"), "w"), indent=1)
    open(os.path.join(PROF, f"{tag}_summary.md"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
