"""Per-kernel summary of an `ncu --set full` report: duration, DRAM bytes and the
physical DRAM fraction against MEASURED_PEAKS.json (6549.4 GB/s measured copy)."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]
UNIT = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1e-3, "msecond": 1e-3, "us": 1e-6,
        "usecond": 1e-6, "ns": 1e-9, "nsecond": 1e-9}


def main(path, peak=6549.4):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for row in rows[2:]:
        d, u = dict(zip(hdr, row)), dict(zip(hdr, units))
        name = d["Kernel Name"].split("(")[0].replace("(anonymous namespace)::", "")
        val = lambda k: float(d[k].replace(",", "")) * UNIT.get(u[k], 1.0)  # noqa: E731
        t = val("gpu__time_duration.sum")
        b = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
        print(f"{name}: {t * 1e3:.3f} ms, DRAM {b / 1e6:.1f} MB -> {b / t / 1e9:.0f} GB/s = {b / t / 1e9 / peak:.3f} of "
              f"measured {peak} GB/s")
        for k in KEYS[3:]:
            if k in d:
                print(f"    {k:58s} {d[k]} {u[k]}")


if __name__ == "__main__":
    main(sys.argv[1])
