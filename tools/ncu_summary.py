"""One-page summary of an `ncu --set full` report: per kernel launch, the
duration, DRAM bytes, L2 hit rate, throughputs, tensor-pipe activity and
registers.  usage: python tools/ncu_summary.py report.ncu-rep [iterations]"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def main(rep, iters=None):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for d in rows[2:]:
        if len(d) != len(hdr):
            continue
        print(f"kernel: {d[hdr.index('Kernel Name')][:120]}")
        vals = {}
        for key, label in KEYS:
            if key in hdr:
                i = hdr.index(key)
                vals[key] = (d[i], units[i])
                print(f"  {label:28s} {d[i]:>16s} {units[i]}")
        if iters and "dram__bytes_read.sum" in vals:
            def to_b(v, u):
                return float(v.replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            rd = to_b(*vals["dram__bytes_read.sum"])
            wr = to_b(*vals["dram__bytes_write.sum"])
            print(f"  per iteration ({iters}):      read {rd / iters / 1e6:.1f} MB, write {wr / iters / 1e6:.1f} MB")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else None)
