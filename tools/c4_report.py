"""Render the C4 sweep report from a tools/sweep_window.py log and gpurun_out/c4_ncu_M<M>.csv
(tools/c4_ncu_study.sh) plus the ptxas spill counts of the build.

    python tools/c4_report.py gpurun_out/r02o_c4_sweep.log > profiles/r02_c4_sweep.md
"""
import csv
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")


def spills(M, kn):
    """ptxas spill stores/loads of the paper-path (COUNT = false) instance of kernel kn."""
    txt = open(os.path.join(ROOT, "build", "bosrm", f"demod_m{M}.o.log")).read()
    tail = "ELb0ELb0E" if kn in ("demod_kernel", "demod_wide_kernel") else "ELb0E"
    m = re.search(r"Function properties for _ZN3bos\d+%sILi%d%s\S*\s+(\d+) bytes stack frame, (\d+) bytes spill "
                  r"stores, (\d+) bytes spill loads" % (kn, M, tail), txt)
    return f"{m.group(2)}/{m.group(3)}" if m else "?"


def ncu_rows():
    rows = []
    for fn in sorted(os.listdir(OUT), key=lambda f: int(re.sub(r"\D", "", f) or 0)):
        m = re.match(r"c4_ncu_M(\d+)\.csv$", fn)
        if not m:
            continue
        M = int(m.group(1))
        lines = open(os.path.join(OUT, fn)).read().splitlines()
        hi = [i for i, l in enumerate(lines) if l.startswith('"ID"')]
        if not hi:
            continue
        r = list(csv.reader(lines[hi[0]:]))
        ix = {h: i for i, h in enumerate(r[0])}
        d, name = {}, ""
        for x in r[1:]:
            d[x[ix["Metric Name"]]] = (x[ix["Metric Value"]], x[ix["Metric Unit"]])
            name = x[ix["Kernel Name"]]
        rows.append((M, name, d))
    return rows


def main():
    log = sys.argv[1] if len(sys.argv) > 1 else os.path.join(OUT, "c4_sweep.log")
    sweep = [l for l in open(log).read().splitlines() if l.startswith("|")]
    print("# C4 window sweep — single-B200 roofline study (BASELINE config 4), round 2\n")
    print("2048² frames of the C4 generator (diffusion phase, t = 60 + 30k s, 10 dB). Throughput:")
    print("`python tools/sweep_window.py --sizes 8,…,32 --frames 8 --parity-px 16384` (8 flow frames per")
    print("launch against the demodulated reference, CUDA events, 3 reps, inputs resident; parity =")
    print("16,384 sampled pixels of the last frame vs the FP64 oracle). Flop model and peak as in")
    print("bench.py (FP32 FMA, 148 SM × 128 lanes × 2 × 1965 MHz = 74.45 TFLOP/s), iteration counts")
    print("measured, for the kernel that runs each M (bench.path_flops): the register strip kernel")
    print("(R_y slid by one row per pixel) for M ≤ 10, 12, 13; the implicit-power-iteration strip")
    print("kernel (no R_y: y = Γ_w(Γ_w^H u)) for M = 11, 14…32.\n")
    print("\n".join(sweep))
    print("\nPipe / occupancy counters, one 2048² frame per M (`tools/c4_ncu_study.sh`: ncu --metrics,")
    print("second launch of `tools/one_launch.py`, --clock-control none; ptxas spills from the build")
    print("log). \"warp inst / px\": warp instructions per pixel (a warp instruction covers 32 pixels).")
    print("DRAM writes land in L2 within a 2-frame launch.\n")
    print("| M | kernel | time (ms, 2 frames) | FMA pipe % | ALU pipe % | XU (MUFU) inst % | FP64 pipe % | "
          "issue active % | warps active % | regs | spill st/ld B (ptxas) | DRAM read B/px | warp inst / px |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    for M, name, d in ncu_rows():
        def g(k):
            try:
                return float(d.get(k, ("n/a", ""))[0].replace(",", ""))
            except ValueError:
                return float("nan")
        t, tu = g("gpu__time_duration.sum"), d["gpu__time_duration.sum"][1]
        tms = t / 1e6 if tu in ("ns", "nsecond") else (t / 1e3 if tu in ("us", "usecond") else t)
        v, u = d["dram__bytes_read.sum"]
        rb = float(v.replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
        px = 2 * 2048 * 2048
        kn = re.search(r"(demod_\w+kernel)", name).group(1)
        print(f"| {M} | {kn} | {tms:.2f} | "
              f"{g('sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active'):.1f} | "
              f"{g('sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active'):.1f} | "
              f"{g('sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active'):.1f} | "
              f"{g('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active'):.1f} | "
              f"{g('sm__issue_active.avg.pct_of_peak_sustained_elapsed'):.1f} | "
              f"{g('sm__warps_active.avg.pct_of_peak_sustained_active'):.1f} | "
              f"{int(g('launch__registers_per_thread'))} | {spills(M, kn)} | {rb / px:.1f} | "
              f"{g('smsp__inst_executed.sum') / px:.0f} |")
    print(sys.stdin.read() if not sys.stdin.isatty() else "")


if __name__ == "__main__":
    main()
