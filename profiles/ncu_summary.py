"""Per-launch table of an ncu --set full report (DRAM traffic, HBM fraction,
fp64 / DMMA pipe activity, IPC), the format of profiles/r1_kernel_roofline.txt.

    ncu -i prof.ncu-rep --page raw --csv > raw.csv
    python profiles/ncu_summary.py raw.csv [hbm_gbs]
"""
import csv
import sys

COLS = {
    "us": "gpu__time_duration.sum",
    "rd": "dram__bytes_read.sum",
    "wr": "dram__bytes_write.sum",
    "fp64": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "dmma": "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "ipc": "sm__inst_executed.avg.per_cycle_active",
}
SCALE = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "nsecond": 1e-3, "usecond": 1.0, "us": 1.0,
         "msecond": 1e3, "ms": 1e3, "ns": 1e-3}


def main(path, hbm=6545.6):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    idx = {k: hdr.index(v) for k, v in COLS.items()}
    kname = hdr.index("Kernel Name")
    print(f"{'kernel':40s} {'us':>8s} {'rd MB':>8s} {'wr MB':>8s} {'GB/s':>7s} {'%HBM':>6s} "
          f"{'fp64%':>6s} {'dmma%':>6s} {'IPC':>5s}")
    for r in rows[2:]:
        def val(k):
            x = r[idx[k]].replace(",", "")
            return float(x) * SCALE.get(units[idx[k]], 1.0) if k in ("us", "rd", "wr") else float(x)
        us, rd, wr = val("us"), val("rd"), val("wr")
        gbs = (rd + wr) / us * 1e3 if us > 0 else 0.0
        name = r[kname].split("(")[0].replace("void ", "").replace("ttb::", "").replace(", ", ",")[:40]
        print(f"{name:40s} {us:8.1f} {rd:8.1f} {wr:8.1f} {gbs:7.0f} {100 * gbs / hbm:6.1f} "
              f"{val('fp64'):6.1f} {val('dmma'):6.1f} {val('ipc'):5.2f}")


if __name__ == "__main__":
    main(sys.argv[1], *(float(a) for a in sys.argv[2:3]))
