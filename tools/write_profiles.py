"""Turn the ncu outputs of a GPU run into the committed evidence under profiles/.

    python tools/write_profiles.py --round r01 --launches gpurun_out/launches.csv \
        --rep gpurun_out/prof_expand_L3.ncu-rep --plain gpurun_out/p.log

Writes profiles/<round>_launches.csv (the raw launch list), profiles/<round>_launch_summary.md
(per-kernel totals and shares of the BFS kernels), profiles/<round>_expand_L3.txt (key metrics of
the captured k_expand launch) and profiles/expand_traffic.json (its DRAM bytes per launch, read by
bench.py for roofline.traffic).
"""
import argparse
import collections
import csv
import io
import json
import os
import re
import shutil
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")
BUILD = {"k_count", "k_scatter", "k_kron_generate", "k_keys_to_rows", "k_keys_to_cols", "k_csr_keys", "k_offsets",
         "k_slice", "k_degree_keys", "k_iota2", "k_apply_moves", "k_count_nz_rows", "k_perm_from_sorted", "k_narrow", "k_deg8"}


def launch_summary(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0}
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in data:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-6)
        name = re.sub(r"^void ", "", r[ki]).split("(")[0].split("<")[0].replace("bfs200::", "")
        if (name.startswith("cub::") and "DeviceScan" not in name) or name in BUILD:
            name = "[construction] " + name
        elif name in ("k_mcomp", "k_degree"):
            name = "[outside the timed search] " + name
        tot[name] += v
        cnt[name] += 1
    return tot, cnt


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r01")
    ap.add_argument("--launches")
    ap.add_argument("--rep")
    ap.add_argument("--plain")
    a = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    if a.launches:
        shutil.copy(a.launches, os.path.join(PROF, f"{a.round}_launches.csv"))
        tot, cnt = launch_summary(a.launches)
        bfs = {k: v for k, v in tot.items() if not k.startswith("[")}
        T = sum(bfs.values())
        lines = [f"# {a.round}: ncu launch list (gpu__time_duration.sum, --clock-control none)", "",
                 "One BFS from the first sampled root of the s26 1x1 bench graph (tools/profile_bfs.py --roots 1).",
                 "ncu serialises launches and runs them cold-cache: compare SHARES, not absolute times.", "",
                 "| kernel | launches | total ms | share of BFS kernels |", "|---|---|---|---|"]
        for k, v in sorted(bfs.items(), key=lambda x: -x[1]):
            lines.append(f"| {k} | {cnt[k]} | {v:.3f} | {100 * v / T:.1f}% |")
        lines += ["", f"BFS kernels total: {T:.3f} ms (the timed search: init .. outputs)", "",
                  "Not in the timed search (graph construction; m_comp and root-degree queries):", ""]
        for k, v in sorted(tot.items(), key=lambda x: -x[1]):
            if k.startswith("["):
                lines.append(f"- {k}: {cnt[k]} launches, {v:.3f} ms")
        open(os.path.join(PROF, f"{a.round}_launch_summary.md"), "w").write("\n".join(lines) + "\n")
    if a.rep:
        out = subprocess.run(["python", os.path.join(ROOT, "tools", "ncu_summary.py"), a.rep], capture_output=True,
                             text=True).stdout
        raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        hdr, units = rows[0], rows[1]
        d = [r for r in rows[2:] if "k_expand" in r[hdr.index("Kernel Name")]][0]

        def val(name):
            i = hdr.index(name)
            mul = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(units[i], 1)
            return float(d[i].replace(",", "")) * mul

        stalls = []
        for i, k in enumerate(hdr):
            if "average_warps_issue_stalled" in k and "per_issue_active" in k:
                try:
                    v = float(d[i].replace(",", ""))
                except ValueError:
                    continue
                if v > 0.05:
                    stalls.append((v, k.replace("smsp__average_warps_issue_stalled_", "").replace(
                        "_per_issue_active.ratio", "")))
        units_pct = ["lts__t_tag_requests.avg.pct_of_peak_sustained_elapsed",
                     "lts__t_tag_requests.max.pct_of_peak_sustained_elapsed",
                     "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
                     "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
                     "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
                     "sm__warps_active.avg.pct_of_peak_sustained_active"]
        counts = ["lts__t_requests_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
                  "lts__t_requests_srcunit_tex_op_red.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
                  "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
                  "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum"]
        txt = [f"# {a.round}: ncu --set full capture at the peak level (L3) of one s26 BFS (launches of that level)",
               out, "# k_expand: warp-stall breakdown (cycles per issued instruction, > 0.05)",
               "  " + ", ".join(f"{k}={v:.2f}" for v, k in sorted(stalls, reverse=True)),
               "# k_expand: unit utilisation (%)"]
        txt += [f"  {k} = {d[hdr.index(k)]}" for k in units_pct if k in hdr]
        txt += ["# k_expand: request / sector counts"]
        txt += [f"  {k} = {d[hdr.index(k)]}" for k in counts if k in hdr]
        alg = None
        if a.plain:  # algorithmic bytes of the L3 launch from the plain run (4 B/edge + 40 B/column)
            for line in open(a.plain):
                m = re.match(r"\s+L3: frontier\s+(\d+) edges\s+(\d+)", line)
                if m:
                    alg = 4 * int(m.group(2)) + 40 * int(m.group(1))
                    break
            txt += ["# per-level phase times of the same root (tools/profile_bfs.py, no profiler)", open(a.plain).read()]
        dram = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
        t_ms = float(d[hdr.index("gpu__time_duration.sum")]) * (1e-3 if units[hdr.index("gpu__time_duration.sum")]
                                                                == "usecond" else 1.0)
        if alg:
            txt += [f"# k_expand L3: algorithmic {alg / 1e9:.3f} GB (4 E + 40 F), DRAM {dram / 1e9:.3f} GB "
                    f"(ratio {dram / alg:.3f}), ncu time {t_ms:.3f} ms (cold, serialised)"]
        open(os.path.join(PROF, f"{a.round}_expand_L3.txt"), "w").write("\n".join(txt) + "\n")
        json.dump({"round": a.round, "kernel": "k_expand", "launch": "L3 (peak level), first bench root",
                   "dram_bytes_per_launch": dram, "alg_bytes_per_launch": alg, "alg_definition": "4 E_L + 40 F_L",
                   "ncu_time_ms": t_ms, "source": os.path.basename(a.rep)},
                  open(os.path.join(PROF, "expand_traffic.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
