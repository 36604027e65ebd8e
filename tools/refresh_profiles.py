"""Regenerate the committed round-2 profile summaries from the files a
tools/gpu_prof_r2.sh run merged into gpurun_out/ (bench lines, launch list,
leaf ncu capture, per-kernel roofline tables, config measurements)."""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")


def last_json_line(path):
    return [x for x in open(path) if x.startswith("{")][-1]


def raw_csv(rep, out):
    with open(out, "w") as f:
        subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], stdout=f, stderr=subprocess.DEVNULL, check=True)


def main(note):
    open(os.path.join(P, "r2_bench.json"), "w").write(last_json_line(os.path.join(G, "r2_bench.log")))
    open(os.path.join(P, "r2_bench_reference.json"), "w").write(last_json_line(os.path.join(G, "r2_bench_reference.log")))
    for f in ("r2_launches.csv", "r2_configs.txt"):
        open(os.path.join(P, f), "w").write(open(os.path.join(G, f)).read())
    summ = subprocess.run([sys.executable, os.path.join(P, "summarize_launches.py"), os.path.join(P, "r2_launches.csv")],
                          capture_output=True, text=True, check=True).stdout
    open(os.path.join(P, "r2_launches_summary.txt"), "w").write(
        "# ncu --metrics gpu__time_duration.sum --clock-control none, python profiles/round_once.py 2 (two cfg3 "
        "roundings + input generation): cold-cache, serialised launch times\n" + summ)
    raw_csv(os.path.join(G, "r2_leaf.ncu-rep"), "/tmp/leaf.csv")
    rows = list(csv.reader(open("/tmp/leaf.csv")))
    hdr, units, r = rows[0], rows[1], rows[2]
    sc = {"Mbyte": 1.0, "Gbyte": 1e3, "Kbyte": 1e-3, "byte": 1e-6, "us": 1.0, "usecond": 1.0, "ms": 1e3,
          "msecond": 1e3, "ns": 1e-3}

    def g(name):
        i = hdr.index(name)
        return float(r[i].replace(",", "")) * sc.get(units[i], 1.0)

    d = {"kernel": r[hdr.index("Kernel Name")],
         "capture": "ncu --set full --clock-control none --import-source on -k regex:tsqr_leaf -s 30 -c 1 python "
                    "profiles/round_once.py 2",
         "launch": "one sweep-2 leaf: H(X_n)^T panel, 240000 x 60 (rows = 8000 slices x rank 30), grid 148 x 256",
         "gpu_time_us": g("gpu__time_duration.sum"), "dram_read_MB": g("dram__bytes_read.sum"),
         "dram_write_MB": g("dram__bytes_write.sum"), "algorithmic_MB": 230.4,
         "registers_per_thread": g("launch__registers_per_thread"),
         "fp64_pipe_active_pct": g("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
         "dmma_pipe_active_pct": g("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active"),
         "ipc": g("sm__inst_executed.avg.per_cycle_active"), "warp_instructions": g("smsp__inst_executed.sum"),
         "note": note}
    pre, suf = "smsp__average_warps_issue_stalled_", "_per_issue_active.ratio"
    st = {h[len(pre):-len(suf)]: float(r[i].replace(",", "")) for i, h in enumerate(hdr)
          if h.startswith(pre) and h.endswith(suf)}
    d["stalls_per_issue"] = dict(sorted(st.items(), key=lambda kv: -kv[1])[:8])
    json.dump(d, open(os.path.join(P, "r2_leaf_ncu.json"), "w"), indent=1)
    out = ["# round-2 final captures (ncu --set full --clock-control none): Gram / Hadamard "
           "(profiles/kernel_roofline.py), one apply-product launch of a 480000 x 60 panel with k = 60 "
           "(tools/tsqr_bench.py), one sweep-1 R-fold of cfg3\n"]
    for rep in ("r2_kr", "r2_product", "r2_fold"):
        path = os.path.join(G, rep + ".ncu-rep")
        if not os.path.exists(path):
            continue
        raw_csv(path, "/tmp/kr.csv")
        out.append(subprocess.run([sys.executable, os.path.join(P, "ncu_summary.py"), "/tmp/kr.csv"],
                                  capture_output=True, text=True, check=True).stdout)
    open(os.path.join(P, "r2_kernel_roofline.txt"), "w").write("".join(out))
    b = json.loads(last_json_line(os.path.join(G, "r2_bench.log")))
    print(b["ms_per_step"], b["value"], b["e2e"]["ms_per_step"], b["e2e"]["pageable"]["ms_per_step"],
          b["roofline"]["frac"], b["step_roofline"]["kernel_ms"])
    print(open(os.path.join(P, "r2_launches_summary.txt")).read())


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "")
