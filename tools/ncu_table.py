"""Summarise an `ncu --page raw --csv` export: per kernel (averaged over its launches)
time, DRAM throughput, FP64 / DMMA pipe utilisation, warps active and the top stall.
Usage: python tools/ncu_table.py export.csv [more.csv ...]"""
import collections
import csv
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "nsecond": 1e-9}


def load(path):
    rows = list(csv.reader(open(path)))
    h, u = rows[0], rows[1]

    def val(r, k):
        if k not in h:
            return 0.0
        x = r[h.index(k)].replace(",", "")
        try:
            return float(x) * SCALE.get(u[h.index(k)], 1.0)
        except ValueError:
            return 0.0

    out = []
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "").replace("bfly::", "")
        st = [(k, val(r, k)) for k in h if k.startswith("smsp__average_warps_issue_stalled")
              and k.endswith("per_issue_active.ratio")]
        top = max(st, key=lambda x: x[1])[0].replace("smsp__average_warps_issue_stalled_", "").replace(
            "_per_issue_active.ratio", "") if st else "-"
        t = val(r, "gpu__time_duration.sum")
        dram = val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")
        pct = lambda k: float(r[h.index(k)]) if k in h and r[h.index(k)] not in ("", "n/a") else 0.0  # noqa: E731
        out.append((name, t, dram, pct("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
                    pct("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active"),
                    pct("sm__warps_active.avg.pct_of_peak_sustained_active"), top))
    return out


def main():
    agg = collections.OrderedDict()
    for path in sys.argv[1:]:
        for rec in load(path):
            agg.setdefault(rec[0], []).append(rec)
    print("| kernel | launches | ms / launch | DRAM TB/s | FP64 pipe % | DMMA pipe % | warps active % | top stall |")
    print("|---|---|---|---|---|---|---|---|")
    for name, v in agg.items():
        n = len(v)
        t = sum(x[1] for x in v) / n
        bw = sum(x[2] / x[1] for x in v if x[1]) / n / 1e12
        print(f"| `{name}` | {n} | {t * 1e3:.2f} | {bw:.2f} | {sum(x[3] for x in v) / n:.1f} | "
              f"{sum(x[4] for x in v) / n:.1f} | {sum(x[5] for x in v) / n:.1f} | {v[0][6]} |")


if __name__ == "__main__":
    main()
