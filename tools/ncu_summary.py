"""Summarise ncu reports into markdown for profiles/.

    python tools/ncu_summary.py REPORT.ncu-rep [--title T] [--algo-flop F] [--algo-bytes B]

Prints launch metrics (duration, throughput %, occupancy, DRAM bytes),
the SASS instruction mix and the warp-stall breakdown.  Reads reports only
(no GPU needed).
"""
import argparse
import collections
import csv
import io
import subprocess
import sys

NCU = "/usr/local/cuda/bin/ncu"


def ncu_csv(rep, *args):
    out = subprocess.run([NCU, "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def details(rep):
    rows = ncu_csv(rep, "--page", "details")
    hdr = rows[0]
    res = collections.OrderedDict()
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        res[d.get("Metric Name")] = (d.get("Metric Value"), d.get("Metric Unit"), d.get("Kernel Name"))
    return res


def raw(rep):
    rows = ncu_csv(rep, "--page", "raw")
    return {h: (v, u) for h, v, u in zip(rows[0], rows[2], rows[1])}


def sass(rep):
    rows = ncu_csv(rep, "--page", "source", "--print-source", "sass")
    hdr = rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    data = [r for r in rows[2:] if len(r) == len(hdr)]
    mix, stalls = collections.Counter(), collections.Counter()
    tot, tot_s = 0.0, 0.0
    for r in data:
        toks = r[idx["Source"]].split()
        op = toks[0] if toks else "?"
        if op.startswith("@") and len(toks) > 1:
            op = toks[1]
        op = op.split(".")[0]
        n = float(r[idx["Instructions Executed"]] or 0)
        mix[op] += n
        tot += n
        for h in hdr:
            if h.startswith("stall_") and "Not Issued" not in h:
                try:
                    stalls[h] += float(r[idx[h]] or 0)
                    tot_s += float(r[idx[h]] or 0)
                except ValueError:
                    pass
    return mix, tot, stalls, tot_s


def fnum(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return float("nan")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--title", default=None)
    ap.add_argument("--algo-flop", type=float, default=None,
                    help="algorithmic FLOP of the profiled launch")
    args = ap.parse_args()
    d = details(args.report)
    rw = raw(args.report)
    kname = next(iter(d.values()))[2]
    print(f"### {args.title or kname}\n")
    print(f"kernel: `{kname}`\n")
    keys = ["Duration", "Grid Size", "Block Size", "Registers Per Thread",
            "Dynamic Shared Memory Per Block", "Achieved Occupancy", "Executed Ipc Active",
            "Issue Slots Busy", "Compute (SM) Throughput", "L1/TEX Cache Throughput",
            "L2 Cache Throughput", "DRAM Throughput", "L1/TEX Hit Rate", "L2 Hit Rate"]
    print("| metric | value |\n|---|---|")
    for k in keys:
        if k in d:
            print(f"| {k} | {d[k][0]} {d[k][1]} |")
    rb = fnum(rw.get("dram__bytes_read.sum", ("nan",))[0])
    wb = fnum(rw.get("dram__bytes_write.sum", ("nan",))[0])
    ru = rw.get("dram__bytes_read.sum", ("", ""))[1]
    print(f"| dram__bytes_read.sum + write.sum | {rb} + {wb} {ru} |")
    for k in ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
              "l1tex__m_xbar2l1tex_read_bytes.sum", "lts__t_sectors_srcunit_tex.sum"):
        if k in rw:
            print(f"| {k} | {rw[k][0]} {rw[k][1]} |")
    if args.algo_flop and "Duration" in d:
        dur = fnum(d["Duration"][0])
        unit = d["Duration"][1]
        sec = dur * {"ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1.0}.get(unit, 1e-3)
        print(f"| algorithmic TFLOP/s (cold, under ncu) | {args.algo_flop / sec / 1e12:.2f} |")
    mix, tot, stalls, tot_s = sass(args.report)
    print("\nSASS instruction mix (warp instructions executed):\n")
    print("| op | share |\n|---|---|")
    for op, n in mix.most_common(10):
        print(f"| {op} | {100 * n / tot:.1f}% |")
    print("\nwarp stall samples:\n")
    print("| reason | share |\n|---|---|")
    for h, n in stalls.most_common(8):
        print(f"| {h[6:]} | {100 * n / max(tot_s, 1):.1f}% |")
    print()


if __name__ == "__main__":
    sys.exit(main())
