"""Copy the evidence a tools/round2_final2.sh run left in gpurun_out/ into profiles/ (bench
lines, launch lists and their summaries, DRAM traffic of the multiply, the column gather and
the panel generator, the config-5 host timeline):  python tools/refresh_profiles.py"""
import csv
import os
import shutil
import subprocess
import sys

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
head = subprocess.run(["git", "rev-parse", "--short", "HEAD"], cwd=ROOT, capture_output=True, text=True).stdout.strip()


def table(path):
    return subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_table.py"), path],
                          capture_output=True, text=True).stdout


shutil.copy(os.path.join(G, "rf_bench.json"), os.path.join(P, "round2_bench_n1.jsonl"))
open(os.path.join(P, "round2_bench_reference.jsonl"), "w").write(open(os.path.join(G, "rf_ref.log")).read().strip().splitlines()[-1] + "\n")
shutil.copy(os.path.join(G, "rf_launches.csv"), os.path.join(P, "round2_launches.csv"))
open(os.path.join(P, "round2_launch_summary.txt"), "w").write(
    f"# round 2 (head {head}): bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-eigh under ncu (gpu__time_duration.sum, --clock-control none), our kernels\n"
    "# 4 config-4 merges (3 warm-up + 1 timed) -> divide by 4; ncu serialises kernels, so the leaf up-level (capped grid, normally beside the construction) is not overlapped here\n"
    + table(os.path.join(G, "rf_launches.csv")))
subprocess.run([sys.executable, os.path.join(ROOT, "tools", "traffic_json.py"), os.path.join(G, "rf_mult.csv"),
                os.path.join(P, "round2_multiply_dram_launches.csv")], check=True, capture_output=True)
open(os.path.join(P, "round2_cfg5_launch_summary.txt"), "w").write(
    f"# round 2 (head {head}): tools/eigh_prof.py 5 65536 under ncu (gpu__time_duration.sum): TWO full solves of BASELINE config 5 (N = 65536) -> divide by 2\n"
    + table(os.path.join(G, "rf_cfg5.csv")))
shutil.copy(os.path.join(G, "rf_cfg5_host.txt"), os.path.join(P, "round2_cfg5_host_timeline.txt"))


def load(path):
    rows, hdr, per = list(csv.reader(open(path))), None, {}
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            e = per.setdefault(int(d["ID"]), {"name": d["Kernel Name"], "grid": d["Grid Size"]})
            e[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    return [per[i] for i in sorted(per)]


out = [f"# round 2 (head {head}): DRAM traffic of the HBM-bound kernels (ncu dram__bytes_read/write.sum, gpu__time_duration.sum; --clock-control none)",
       "# peak: measured copy bandwidth 6534 GB/s (MEASURED_PEAKS.json)",
       "# kernel  grid  ms  read_GB  write_GB  GB/s  frac_of_peak"]
for title, path, key, sel in (
        ("## wave_gather_kernel<2, 4>, the 12 recursion depths of one config-5 solve (deepest first)",
         "rf_cfg5_gather.csv", "wave_gather", slice(-12, None)),
        ("## gen_panel_rows_kernel<8>, panel row chunks of the config-4 sample (8192 x 32768 doubles each)",
         "rf_genpanel.csv", "gen_panel_rows", slice(0, 8))):
    out.append(title)
    for e in [x for x in load(os.path.join(G, path)) if key in x["name"]][sel]:
        t, r, w = e["gpu__time_duration.sum"] / 1e9, e["dram__bytes_read.sum"], e["dram__bytes_write.sum"]
        out.append(f"{key} {e['grid']:>14} {t * 1e3:8.3f} {r / 1e9:8.3f} {w / 1e9:8.3f} {(r + w) / t / 1e9:8.1f} {(r + w) / t / 6534e9:6.3f}")
open(os.path.join(P, "round2_hbm_kernels.txt"), "w").write("\n".join(out) + "\n")
print("profiles refreshed at", head)
