"""Summarise ncu --set full reports (raw page) into a markdown table.

  python scripts/ncu_summary.py gpurun_out/t_gate_up.ncu-rep ... > profiles/r01/ncu_summary.md
"""
import csv
import io
import subprocess
import sys

WANT = [
    ("gpu__time_duration.sum", "dur"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor_%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%"),
    ("lts__t_bytes.sum", "l2_bytes"),
    ("launch__grid_size", "grid"),
    ("launch__registers_per_thread", "regs"),
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1,
         "msecond": 1e3, "%": 1, "": 1, "register/thread": 1}


def rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    for line in r[2:]:
        rec = {"kernel": line[hdr.index("Kernel Name")][:60]}
        for metric, key in WANT:
            if metric in hdr:
                i = hdr.index(metric)
                try:
                    v = float(line[i].replace(",", "")) * SCALE.get(units[i], 1)
                except ValueError:
                    v = float("nan")
                rec[key] = v
        yield rec


print("| report | kernel | grid | dur us | DRAM rd+wr MB | DRAM GB/s | DRAM % | tensor % | L2 MB |")
print("|---|---|---|---|---|---|---|---|---|")
for path in sys.argv[1:]:
    for rec in rows(path):
        mb = (rec.get("dram_rd", 0) + rec.get("dram_wr", 0)) / 1e6
        gbs = mb * 1e6 / (rec["dur"] * 1e-6) / 1e9 if rec.get("dur") else 0
        print(f"| {path.split('/')[-1]} | {rec['kernel']} | {rec.get('grid', 0):.0f} | "
              f"{rec.get('dur', 0):.1f} | {mb:.1f} | {gbs:.0f} | {rec.get('dram_%', 0):.1f} | "
              f"{rec.get('tensor_%', 0):.1f} | {rec.get('l2_bytes', 0) / 1e6:.1f} |")
