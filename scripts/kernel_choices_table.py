"""ncu counters of scripts/kernel_choices.py -> profiles/r02_kernel_choices.md.
usage: python scripts/kernel_choices_table.py <ncu csv> <driver stdout> <out.md> [peak GB/s]

Per launch: time, algorithmic GB/s (read + write of the described bytes) and
its fraction of the copy peak, DRAM bytes per algorithmic byte, and sector
efficiency = useful bytes / (32 B x global load / store sectors,
l1tex__t_sectors_pipe_lsu_mem_global_op_{ld,st}); TMA launches move data
outside the LSU pipe, so they have none."""
import csv
import sys
from collections import OrderedDict

KERNELS = ("k_words", "k_smallrow", "k_tma", "k_shift", "k_runs", "k_batch", "k_job")


def main(csv_path, log_path, out_path, peak=6547.2):
    rows = OrderedDict()
    with open(csv_path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if not any(k in r["Kernel Name"] for k in KERNELS):
            continue
        key = r["ID"]
        d = rows.setdefault(key, {"kernel": r["Kernel Name"].split("(")[0]})
        try:
            d[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
        except ValueError:
            d[r["Metric Name"]] = r["Metric Value"]
    labels = [ln.rstrip("\n").split("\t") for ln in open(log_path) if ln[:1].isdigit()]
    launches = list(rows.values())
    if len(launches) != len(labels):
        raise SystemExit(f"{len(launches)} launches vs {len(labels)} labels")
    out = ["# Every automatic kernel choice under ncu (round 2)", "",
           "Source: `scripts/kernel_choices.py`, one launch per case, each after an L2 flush. The counter pass",
           "is `scripts/gpu_kernel_choices.sh`, the CSV is `profiles/r02_kernel_choices.csv`, and this table",
           "comes from `scripts/kernel_choices_table.py`. ncu replays each kernel with caches flushed and",
           "serialised, so the times are cold.", "",
           "Columns:",
           "* alg. GB/s = read + write of the described bytes / time;",
           f"* % peak = alg. GB/s / {peak} (measured copy peak, MEASURED_PEAKS.json);",
           "* DRAM / alg. = (DRAM read + write bytes) / algorithmic bytes (1.0 = no wasted traffic);",
           "* ld / st eff. = sector efficiency of the global loads / stores: useful bytes (half the",
           "  algorithmic bytes on each side) / (32 B x l1tex__t_sectors_pipe_lsu_mem_global_op_{ld,st}),",
           "  in % (LSU path only; TMA moves data outside it, so those launches show `-`).", "",
           "| case | chosen | kernel | us | alg. GB/s | % peak | DRAM GB/s | DRAM / alg. | ld eff. % | st eff. % |",
           "|---|---|---|---:|---:|---:|---:|---:|---:|---:|"]
    for (i, label, nbytes, chosen), m in zip(labels, launches):
        us = m.get("gpu__time_duration.sum", 0) / 1e3
        alg = int(nbytes)
        dram = m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
        gbs = alg / (us * 1e3) if us else 0
        dgbs = dram / (us * 1e3) if us else 0

        def eff(name):
            v = m.get(name)
            return f"{100 * (alg / 2) / (32 * v):.1f}" if isinstance(v, float) and v > 0 else "-"

        out.append(f"| {label} | {chosen} | `{m['kernel'][:28]}` | {us:.1f} | {gbs:.0f} | {100 * gbs / peak:.1f} | "
                   f"{dgbs:.0f} | {dram / alg:.2f} | "
                   f"{eff('l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum')} | "
                   f"{eff('l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum')} |")
    out.append("")
    open(out_path, "w").write("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], *(float(x) for x in sys.argv[4:]))
