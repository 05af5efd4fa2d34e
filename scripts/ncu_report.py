"""Summarise an ncu --set full report: key raw metrics + top stall sites (SASS).
usage: python scripts/ncu_report.py REP.ncu-rep [N_TOP]"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg.per_second",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    r = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    h, units, row = r[0], r[1], r[2]
    for k in KEYS:
        if k in h:
            i = h.index(k)
            print(f"{k:70s} {row[i]} {units[i]}")
    src = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "sass"))))
    hh = src[1]
    i_s, i_src = hh.index("Warp Stall Sampling (All Samples)"), hh.index("Source")
    data = [x for x in src[2:] if len(x) > i_s and x[i_s].isdigit()]
    tot = sum(int(x[i_s]) for x in data)
    print(f"stall samples {tot}")
    for x in sorted(data, key=lambda x: -int(x[i_s]))[:ntop]:
        print(f"{100 * int(x[i_s]) / tot:5.1f}%  {x[0][-5:]}  {x[i_src].strip()[:100]}")


if __name__ == "__main__":
    main()
