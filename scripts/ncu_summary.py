"""Key metrics of ncu --set full reports (one launch each) as CSV rows."""
import csv
import io
import subprocess
import sys

UNIT = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "byte": 1e-6, "Kbyte": 1e-3,
        "Mbyte": 1.0, "Gbyte": 1e3}
KEYS = {
    "duration_us": ("gpu__time_duration.sum", None),
    "dram_read_MB": ("dram__bytes_read.sum", None),
    "dram_write_MB": ("dram__bytes_write.sum", None),
    "dram_pct_peak": ("dram__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "sm_issue_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "tensor_pipe_pct": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "fma_pipe_pct": ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", 1),
    "xu_pipe_pct": ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", 1),
    "regs": ("launch__registers_per_thread", 1),
    "grid": ("launch__grid_size", 1),
    "block": ("launch__block_size", 1),
}


def read(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for row in rows[2:]:
        d = {"kernel": row[h.index("Kernel Name")].split("(")[0]}
        for k, (m, sc) in KEYS.items():
            if m in h:
                i = h.index(m)
                if sc is None:
                    sc = UNIT.get(units[i], 1.0)
                try:
                    d[k] = round(float(row[i].replace(",", "")) * sc, 3)
                except ValueError:
                    d[k] = row[h.index(m)]
        res.append(d)
    return res


if __name__ == "__main__":
    w = None
    for rep in sys.argv[1:]:
        for d in read(rep):
            if w is None:
                w = csv.DictWriter(sys.stdout, fieldnames=list(d.keys()))
                w.writeheader()
            w.writerow(d)
