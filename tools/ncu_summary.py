#!/usr/bin/env python
"""Summarise the round's ncu outputs (tools/profile_round.sh) into markdown tables.
usage: python tools/ncu_summary.py gpurun_out [--hbm-peak 6533.8]"""
import collections
import csv
import io
import subprocess
import sys


def launch_table(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.OrderedDict()
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            k = d["Kernel Name"].split("(")[0].replace("ozr::", "").replace("(anonymous namespace)::", "")
            v = float(d["Metric Value"].replace(",", ""))
            unit = d.get("Metric Unit", "ns")
            v = v * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}.get(unit, 1e-6)
            a = agg.setdefault(k, [0, 0.0])
            a[0] += 1
            a[1] += v
    tot = sum(v[1] for v in agg.values())
    out = ["| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| {k} | {c} | {t:.2f} | {t / tot:.3f} |")
    return "\n".join(out), agg


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "sm__inst_executed_pipe_tensor_op_imma.avg.pct_of_peak_sustained_active",
           "launch__registers_per_thread", "launch__grid_size", "smsp__cycles_active.avg.pct_of_peak_sustained_elapsed",
           "sm__cycles_elapsed.avg.per_second", "lts__t_sector_hit_rate.pct"]


def raw(rep):
    import os
    csvp = rep.replace(".ncu-rep", "_raw.csv")  # exported on the GPU box (ncu -i … --page raw --csv)
    if os.path.exists(csvp):
        txt = open(csvp).read()
    else:
        txt = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True)
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        out.append((d, u))
    return out


def num(d, u, k):
    v = d.get(k)
    if v in (None, "", "n/a"):
        return None
    v = float(v.replace(",", ""))
    unit = u.get(k, "")
    scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "KB": 1e3, "MB": 1e6, "GB": 1e9,
             "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3,
             "cycle/nsecond": 1e3, "cycle/usecond": 1.0, "Ghz": 1e3, "Mhz": 1.0}.get(unit, 1.0)
    return v * scale


def full_table(rep, hbm_peak):
    out = ["| kernel | grid | ms | DRAM rd+wr GB | achieved GB/s | % of HBM peak | dram % (ncu) | SM % | tensor pipe % | regs |",
           "|---|---|---|---|---|---|---|---|---|---|"]
    for d, u in raw(rep):
        name = d.get("Kernel Name", "?").split("(")[0].replace("ozr::", "").replace("(anonymous namespace)::", "")
        ms = num(d, u, "gpu__time_duration.sum")
        rb = num(d, u, "dram__bytes_read.sum") or 0.0
        wb = num(d, u, "dram__bytes_write.sum") or 0.0
        gb = (rb + wb) / 1e9
        gbs = gb / (ms / 1e3) if ms else 0.0
        f = lambda k: (f"{num(d, u, k):.1f}" if num(d, u, k) is not None else "-")  # noqa: E731
        out.append(f"| {name} | {d.get('launch__grid_size', '?')} | {ms:.3f} | {gb:.3f} | {gbs:.0f} | "
                   f"{100 * gbs / hbm_peak:.1f} | {f('dram__throughput.avg.pct_of_peak_sustained_elapsed')} | "
                   f"{f('sm__throughput.avg.pct_of_peak_sustained_elapsed')} | "
                   f"{f('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed')} | "
                   f"{d.get('launch__registers_per_thread', '?')} |")
    return "\n".join(out)


def algorithmic_bytes_per_element(name, sw):
    """Algorithmic bytes per element of an n x n launch for the sweep plan `sw` (the bench line's
    "sweep" dict: kX, kR, kE, planes_V/W/U = group planes recombined per element); None if not an HBM kernel."""
    kx, kr, ke = sw["kX"], sw["kR"], sw["kE"]
    table = {"k_x1_split": 8 + 8 + kx, "k_x1_split_v": 8 + 8 + kx, "k_colmax": 8,
             "k_recombine_V": 4 * sw.get("planes_V", 0) + 8 + 16, "k_split_res": 24 + kr,
             "k_recombine_E": 4 * sw.get("planes_W", 0) + 8, "k_final": 4 * sw.get("planes_U", 0) + 8 + 8 + 8,
             "k_transpose_i8": 2 * kx, "k_transpose_i8_v": 2 * kx, "k_split_fixed(E')": 8 + ke,
             "k_split_fixed(A)": 8 + sw.get("kA_split", 15)}
    base = name.split("<")[0].replace("void ", "").replace("unnamed>::", "").strip()
    return table.get(base)


def algorithmic_table(rep, sw, n, hbm_peak):
    out = ["| kernel | ms (ncu) | algorithmic bytes/element | algorithmic GB | algorithmic GB/s | % of HBM peak |",
           "|---|---|---|---|---|---|"]
    seen_x1 = False
    for d, u in raw(rep):
        name = d.get("Kernel Name", "?").split("(")[0].replace("ozr::", "").replace("(anonymous namespace)::", "")
        seen_x1 = seen_x1 or "x1_split" in name
        if "split_fixed" in name:  # the A split (once per call) precedes the sweep's X̂ split; the Ẽ' split follows it
            name = name.replace("k_split_fixed", "k_split_fixed(E')" if seen_x1 else "k_split_fixed(A)")
        b = algorithmic_bytes_per_element(name, sw)
        ms = num(d, u, "gpu__time_duration.sum")
        if b is None or not ms:
            continue
        gb = b * n * n / 1e9
        gbs = gb / (ms / 1e3)
        out.append(f"| {name} | {ms:.3f} | {b:.1f} | {gb:.3f} | {gbs:.0f} | {100 * gbs / hbm_peak:.1f} |")
    return "\n".join(out)


if __name__ == "__main__":
    d = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
    peak = 6533.8  # fallback: the round-1 measured copy peak
    try:
        import json
        import os
        peak = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        pass
    if "--hbm-peak" in sys.argv:
        peak = float(sys.argv[sys.argv.index("--hbm-peak") + 1])
    t, _ = launch_table(f"{d}/launches.csv")
    print("## Launch list\n\n" + t + "\n")
    if "--bench" in sys.argv:  # algorithmic bytes from the bench line's sweep plan (n x n launches, 1 GPU)
        import json
        line = [ln for ln in open(sys.argv[sys.argv.index("--bench") + 1]) if ln.startswith("{")][-1]
        bj = json.loads(line)
        try:
            print("## hbm_full, algorithmic bytes\n\n" + algorithmic_table(f"{d}/hbm_full.ncu-rep", bj["sweep"],
                                                                           bj["config"]["n"], peak) + "\n")
        except Exception as e:
            print(f"## algorithmic: {e}\n")
    for rep in ("gemm_full", "hbm_full"):
        try:
            print(f"## {rep}\n\n" + full_table(f"{d}/{rep}.ncu-rep", peak) + "\n")
        except Exception as e:
            print(f"## {rep}: {e}\n")
