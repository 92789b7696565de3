"""Summarise ncu outputs into profiles/ (tracked).

python profiles/summarize_ncu.py <launches.csv> <full.ncu-rep | raw-page.csv> <tag> <config> ["<launch-list command>"] [multiplies]
writes profiles/<tag>_launches.md, profiles/<tag>_kernels.md and updates profiles/ncu_traffic.json
(per-kernel-class DRAM bytes per launch, read by bench.py as roofline.traffic).
"""
import collections
import csv
import io
import json
import os
import re
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))


def short(name):
    name = name.replace("unsigned long", "u64").replace("uint4", "u128")
    m = re.match(r"(?:void )?([A-Za-z0-9_]+)(<[^>]*>)?", name)
    return (m.group(1) + (m.group(2) or "")) if m else name[:30]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    per = collections.OrderedDict()
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        key = (d["ID"], short(d["Kernel Name"]))
        per.setdefault(key, {})[d["Metric Name"]] = (float(d["Metric Value"].replace(",", "")), d["Metric Unit"])
    return per


def to_unit(v, u, target):
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "msecond": 1e3, "ms": 1e3,
             "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    return v * scale.get(u, 1.0)


def main():
    lpath, rep, tag, cfg = sys.argv[1:5]
    what = sys.argv[5] if len(sys.argv) > 5 else "one warm multiply"
    nmul = int(sys.argv[6]) if len(sys.argv) > 6 else 1   # multiplies covered by the launch list
    per = launches(lpath)
    cls = collections.OrderedDict()
    for (i, k), m in per.items():
        t = to_unit(*m.get("gpu__time_duration.sum", (0, "ns")), "us")
        rb = to_unit(*m.get("dram__bytes_read.sum", (0, "byte")), "byte")
        wb = to_unit(*m.get("dram__bytes_write.sum", (0, "byte")), "byte")
        c = cls.setdefault(k, [0, 0.0, 0.0])
        c[0] += 1
        c[1] += t
        c[2] += rb + wb
    tot = sum(c[1] for c in cls.values())
    out = [f"# ncu launch list, {cfg} ({tag}) -- `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
           f"dram__bytes_write.sum --clock-control none` over {what} (cold-cache, serialised: compare "
           "shares, not absolutes)\n", "| kernel | launches | total us | share | DRAM bytes / launch |", "|---|---|---|---|---|"]
    traffic = {}
    for k, (n, t, b) in sorted(cls.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| {k} | {n} | {t:.1f} | {100 * t / tot:.1f} % | {b / n / 1e6:.1f} MB |")
        traffic[k] = b / n
    out.append(f"| **total** | {sum(c[0] for c in cls.values())} | {tot:.1f} | 100 % | |")
    open(os.path.join(HERE, f"{tag}_launches.md"), "w").write("\n".join(out) + "\n")
    tj = os.path.join(HERE, "ncu_traffic.json")
    allt = json.load(open(tj)) if os.path.exists(tj) else {}
    # bench.py kernel names
    bmap = {"k_fft2<0, 1>": "k_fft<psi>", "k_fft2<0, 0>": "k_fft", "k_fft2<1, 0>": "k_fft<inv>",
            "k_cvt_tile<u64>": "k_cvt_tile<u64>", "k_cvt_tile<u128>": "k_cvt_tile<u128>",
            "k_cvt_stream<u64>": "k_cvt_stream<u64>", "k_cvt_stream<u128>": "k_cvt_stream<u128>"}
    def bname(k):
        if k in bmap:
            return bmap[k]
        if k.startswith("k_ipsi_bs<1") or k.startswith("k_ipsi_bs<true"):
            return "k_ipsi_mcomb"
        if k.startswith("k_ipsi_bs"):
            return "k_ipsi_bs"
        m = re.match(r"(k_cvt_(?:rb|res|tile|stream|top|slab|seam))(?:_tma)?<(u64|u128)", k)
        if m:
            return f"{m.group(1)}<{m.group(2)}>"
        if k.startswith("k_bottom"):
            return "k_bottom"
        m = re.match(r"k_fft2<(\d), (\d)", k)   # k_fft2<INV, PSI, ZS>
        if m:
            return "k_fft<inv>" if m.group(1) == "1" else ("k_fft<psi>" if m.group(2) == "1" else "k_fft")
        return k
    agg = {}
    for k, v in traffic.items():   # per-launch average over template variants of one bench kernel name
        agg.setdefault(bname(k), []).append((cls[k][0], v))
    allt[cfg] = {k: sum(n * v for n, v in lst) / sum(n for n, _ in lst) for k, lst in agg.items()}
    # whole multiply: DRAM bytes and launches over all passes (SURVEY §8(d) "bytes over all passes")
    allt[cfg]["__step_dram_bytes"] = sum(c[2] for c in cls.values()) / nmul
    allt[cfg]["__step_launches"] = sum(c[0] for c in cls.values()) / nmul
    json.dump(allt, open(tj, "w"), indent=1)
    # full capture
    if rep.endswith(".csv"):   # the raw page already exported on the GPU box (`ncu -i … --page raw --csv`)
        raw = open(rep).read()
    else:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, data = rows[0], rows[2:]
    keys = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "DRAM read"),
            ("dram__bytes_write.sum", "DRAM write"), ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
            ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
            ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
            ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
            ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
            ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/smem %"),
            ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
            ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
            ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
            ("launch__registers_per_thread", "regs/thread"),
            ("smsp__inst_executed.sum", "warp instructions")]
    keys = [(k, n) for k, n in keys if k in hdr]
    stall_cols = [(i, h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""))
                  for i, h in enumerate(hdr) if h.startswith("smsp__average_warps_issue_stalled_")
                  and h.endswith("_per_issue_active.ratio")]
    units = dict(zip(hdr, rows[1]))
    lines = [f"# ncu --set full --clock-control none, {cfg} ({tag}): every kernel of one warm multiply "
             "(tools/dev/prof_run.py)\n", "| kernel | grid x block | " + " | ".join(n for _, n in keys) +
             " | top stalls (warp-cycles per issue) |", "|---|---|" + "---|" * len(keys) + "---|"]
    for r in data:
        d = dict(zip(hdr, r))
        vals = [f"{d[k]} {units.get(k, '')}".strip() for k, _ in keys]
        st = sorted(((float(r[i]), n) for i, n in stall_cols if r[i] not in ("", "n/a")), reverse=True)[:4]
        stalls = ", ".join(f"{n} {v:.2f}" for v, n in st)
        lines.append(f"| {short(d['Kernel Name'])} | {d.get('Grid Size', '')} x {d.get('Block Size', '')} | " +
                     " | ".join(vals) + f" | {stalls} |")
    open(os.path.join(HERE, f"{tag}_kernels.md"), "w").write("\n".join(lines) + "\n")
    print("\n".join(out))
    print("\n".join(lines))


if __name__ == "__main__":
    main()
