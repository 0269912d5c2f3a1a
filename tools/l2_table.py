"""Per-launch L2 / DRAM traffic table from an ncu --csv metric log of tools/l2_probe.py
(metrics: gpu__time_duration.sum, lts__t_bytes.sum, lts__t_sectors_op_read.sum,
dram__bytes_read.sum, dram__bytes_write.sum, sm__cycles_elapsed.avg.per_second,
sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed).
usage: python tools/l2_table.py LOG.csv LAYER,OP,... (names of the launches in probe order)"""
import collections
import csv
import sys


def main():
    rows = list(csv.DictReader(l for l in open(sys.argv[1]) if l.startswith('"')))
    names = sys.argv[2].split(",") if len(sys.argv) > 2 else None
    k = collections.OrderedDict()
    for r in rows:
        k.setdefault((int(r["ID"]), r["Kernel Name"].split("<")[0].replace("void ", "")), {})[r["Metric Name"]] = \
            (float(r["Metric Value"].replace(",", "")), r["Metric Unit"])
    print("| # | launch | kernel | us | SM clk GHz | L2->SM read MB | L2 read B/clk/SM | all L2 B/clk (chip) "
          "| DRAM MB | tensor % |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for i, ((lid, kern), m) in enumerate(k.items()):
        v, u = m["gpu__time_duration.sum"]
        t = v * {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}.get(u, 1e-9)
        clk = m["sm__cycles_elapsed.avg.per_second"][0]
        clk *= {"Ghz": 1e9, "GHz": 1e9, "Mhz": 1e6, "MHz": 1e6}.get(m["sm__cycles_elapsed.avg.per_second"][1], 1.0)
        cyc = t * clk
        rd = m["lts__t_sectors_op_read.sum"][0] * 32
        l2 = m["lts__t_bytes.sum"][0] * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(
            m["lts__t_bytes.sum"][1], 1)
        dr = sum(m[x][0] * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(m[x][1], 1)
                 for x in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        ten = m["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"][0]
        nm = names[i] if names and i < len(names) else str(lid)
        print(f"| {i} | {nm} | {kern} | {t * 1e6:.1f} | {clk / 1e9:.2f} | {rd / 1e6:.0f} | {rd / cyc / 148:.1f} | "
              f"{l2 / cyc:.0f} | {dr / 1e6:.0f} | {ten:.1f} |")


if __name__ == "__main__":
    main()
