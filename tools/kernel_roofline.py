"""Per-kernel roofline rows from one profiled step per configuration
(gpurun_out/steps/step_c*.csv, tools/gpu_r2_steps.sh): the kernels' serialised ncu
durations for exactly one bench step, against the algorithmic work of each kernel class
(standard 5 n log2 n per complex FFT line of the lines the kernel transforms, 8 flops per
complex tap of a NUFFT stencil, bytes for the data-movement kernels).  Peaks: the FP32 FFMA
probe of bench.py (72.1 TFLOP/s on these boxes) and MEASURED_PEAKS.json's copy bandwidth.
Writes a markdown table to stdout."""
import collections
import csv
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FP32 = 72.1e12
try:
    HBM = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] * 1e9
except Exception:
    HBM = 6537.3e9


def times(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[1:]:
        try:
            name = r[ki].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
            agg[name] += float(r[vi].replace(",", "")) * 1e-9   # ns -> s
            cnt[name] += 1
        except ValueError:
            pass
    return agg, cnt


def fft(n):
    return 5.0 * n * math.log2(n)


def pick(agg, *prefixes):
    return sum(v for k, v in agg.items() if any(k.startswith(p) for p in prefixes))


def row(out, cfg, kernel, t, work, kind, model):
    if t <= 0:
        return
    if kind == "flop":
        ach, peak, unit = work / t / 1e12, FP32 / 1e12, "TFLOP/s"
    else:
        ach, peak, unit = work / t / 1e9, HBM / 1e9, "GB/s"
    out.append(f"| {cfg} | `{kernel}` | {t * 1e3:.3f} | {ach:.2f} {unit} | {ach / peak:.2f} | {model} |")


def main(d):
    out = ["| config | kernel (class) | ms per step (ncu, serialised) | achieved | fraction of peak | algorithmic work per step |",
           "|---|---|---|---|---|---|"]
    # config 4 / 5: P = 1024, 8192 (f, plane) units; config 3: P = 512, 3072 units
    for c, P, U, ny in ((4, 1024, 32 * 256, 512), (5, 1024, 32 * 256, 512), (3, 512, 24 * 128, 256)):
        p = os.path.join(d, f"step_c{c}.csv")
        if not os.path.exists(p):
            continue
        agg, _ = times(p)
        h = P // 2 + 1
        row(out, c, "k_pa (A: kernel rows)", pick(agg, "k_pa<"), U * h * fft(P), "flop",
            f"{U} units x {h} lines x 5P log2 P")
        row(out, c, "k_pb12 (fused B)", pick(agg, "k_pb12<"), U * (h + P) * fft(P), "flop",
            f"{U} units x ({h} + {P}) lines")
        row(out, c, "k_pc_h (C, Horner)", pick(agg, "k_pc_h<"), U * ny * fft(P), "flop",
            f"{U} units x {ny} lines")
        if c == 3:
            Q = 2 * P
            row(out, c, "k_bluestein_w x pass", pick(agg, "k_bluestein_w<32, 1"),
                U * 256 * 2 * fft(Q), "flop", f"{U} units x 256 rows x 2 FFT(Q = {Q})")
            row(out, c, "k_bluestein_w y pass", pick(agg, "k_bluestein_w<32, 0"),
                U * P * 2 * fft(Q), "flop", f"{U} units x {P} columns x 2 FFT(Q)")
        D = 262144 if c == 4 else (131072 if c == 5 else 65536)
        T, F = 4096, (32 if c != 3 else 24)
        row(out, c, "k_temporal_dft (K1)", pick(agg, "k_temporal_dft"), D * T * 4 + D * F * 8,
            "byte", "D T 4 + D F 8 bytes")
        if c == 5:
            row(out, c, "k_spread (type-1 spreading)", pick(agg, "k_spread"),
                32 * 131072 * 8 * 8 * 8, "flop", "F x L x 8^2 taps x 8 (ES window)")
            m = 2048
            row(out, c, "k_t1_rows + k_t1_cols (type-1 finish)", pick(agg, "k_t1_"),
                32 * (m + m // 2) * fft(m), "flop", f"F x ({m} rows + {m // 2} kept columns) x FFT({m})")
    for c, planes, nodes in ((2, 64, 1), (7, 228, 12)):
        p = os.path.join(d, f"step_c{c}.csv")
        if not os.path.exists(p):
            continue
        agg, cnt = times(p)
        what = "64 planes" if c == 2 else "228 node planes"
        row(out, c, "k_interp2_es8 (type-2 readout, ES window 8 x 8 taps)", pick(agg, "k_interp2"),
            16 * 1_000_000 * nodes * 8 * 8 * 8, "flop",
            f"F x 1e6 voxels x {nodes} grid(s) x 8^2 taps x 8")
        row(out, c, "k_t2_rows_split + k_t2_cols_split (type-2 start: place + fine-grid inverse FFT)",
            pick(agg, "k_t2_"), 16 * planes * (350 + 700) * 2 * fft(350), "flop",
            f"F x {what} x (350 rows + 700 columns) x 2 FFT(350)")
        row(out, c, "k_prop_kernel_rows + k_prop_columns (generic, P = 350: kernel and product spectra)",
            pick(agg, "k_prop_"), 16 * planes * (176 + 176 + 350) * fft(350), "flop",
            f"F x {what} x (176 + 176 + 350) lines x FFT(350)")
        s1 = 16 * (5.0 * 20 * 270 * 270 * math.log2(20 * 270 * 270)
                   + (40 * 540 + 40 * 270) * fft(540) + 270 * 270 * fft(40)
                   + 4 * 270 * fft(270))
        row(out, c, "k_fft_lines (stage 1: 3D kernel FFT, pruned fine-grid FFT, slab 2D transforms)",
            pick(agg, "k_fft_lines"), s1, "flop",
            "F x (FFT3(20 x 270 x 270) + pruned FFT3(40 x 540 x 540 -> 20 x 270 x 270) + 2 FFT2(270^2))")
        row(out, c, "k_spread<16> (3D type-1 spreading, ES 8^3 taps)", pick(agg, "k_spread"),
            16 * 16384 * 8 ** 3 * 8, "flop", "F x L x 8^3 taps x 8")
    p = os.path.join(d, "step_c1.csv")
    if os.path.exists(p):
        agg, _ = times(p)
        P, U = 140, 16 * 64
        row(out, 1, "k_prop_onchip (P = 140: every stage of a unit in shared memory)",
            pick(agg, "k_prop_onchip", "k_onchip_sum"), U * (71 + 71 + 140 + 64) * fft(P), "flop",
            f"{U} units x (71 + 71 + 140 + 64) lines x FFT(140)")
        row(out, 1, "k_spread<16> (type-1 spreading, ES 8^2 taps)", pick(agg, "k_spread"),
            16 * 4096 * 8 * 8 * 8, "flop", "F x L x 8^2 taps x 8")
        row(out, 1, "k_fft_lines (280-point fine grid)", pick(agg, "k_fft_lines", "k_xfft_lines"),
            16 * (280 + 140) * fft(280), "flop", "F x (280 rows + 140 kept columns) x FFT(280)")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "steps"))
