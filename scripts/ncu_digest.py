"""Digest ncu --page raw --csv captures into one line per kernel launch.

usage: python scripts/ncu_digest.py gpurun_out/r02g_*.raw.csv
Columns: duration, DRAM bytes read+write, L2->SM (lts__t_bytes), tensor-pipe active % of
elapsed, SM throughput %, DRAM throughput %, issued IPC.
"""
import csv
import sys

COLS = [("gpu__time_duration.sum", "us", 1e-3),
        ("dram__bytes_read.sum", "MB", 1e-6), ("dram__bytes_write.sum", "MB", 1e-6),
        ("lts__t_bytes.sum", "MB", 1e-6),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "%", 1.0),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "%", 1.0),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "%", 1.0),
        ("sm__inst_executed.avg.per_cycle_active", "ipc", 1.0)]
UNIT = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6,
        "Gbyte": 1e9, "%": 1.0, "": 1.0, "inst/cycle": 1.0}


def digest(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, units = rows[hi], rows[hi + 1]
    out = []
    for r in rows[hi + 2:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        vals = []
        for k, name, scale in COLS:
            if k not in d or d[k] in ("", "n/a"):
                vals.append(None)
                continue
            v = float(d[k].replace(",", "")) * UNIT.get(u.get(k, ""), 1.0)
            vals.append(v * scale)
        name = d["Kernel Name"].replace("void pp::(anonymous namespace)::", "").split("(")[0]
        out.append((name, d.get("Grid Size", ""), vals))
    return out


def main():
    print("kernel | grid | us | DRAM rd MB | DRAM wr MB | L2 MB | tensor % | SM % | DRAM % | IPC")
    for p in sys.argv[1:]:
        print(f"# {p}")
        for name, grid, v in digest(p):
            f = ["-" if x is None else (f"{x:.1f}" if abs(x) >= 10 else f"{x:.3g}") for x in v]
            print(f"{name[:60]} | {grid} | " + " | ".join(f))


if __name__ == "__main__":
    main()
