"""Summarise an ncu report: key metrics per captured launch, and (optionally) the SASS lines with
the most stall samples for one launch.

    python tools/ncu_summary.py REPORT.ncu-rep [--sass LAUNCH_INDEX] [--top N]
"""
import argparse
import csv
import io
import subprocess

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def raw(rep):
    rows = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv"))))
    hdr, units, data = rows[0], rows[1], rows[2:]
    out = []
    for d in data:
        rec = {"name": d[hdr.index("Kernel Name")][:60]}
        for k in KEYS:
            if k in hdr:
                rec[k] = (d[hdr.index(k)], units[hdr.index(k)])
        out.append(rec)
    return out


def sass(rep, idx, top):
    text = ncu("-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--launch-skip", str(idx),
               "--launch-count", "1")
    rows = list(csv.reader(io.StringIO(text)))
    secs, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1], "rows": []}
            secs.append(cur)
        elif cur is not None:
            cur["rows"].append(r)
    s = max(secs, key=lambda x: len(x["rows"]))
    hdr = s["rows"][0]
    data = [r for r in s["rows"][1:] if len(r) == len(hdr)]
    ie, st, src = (hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)"),
                   hdr.index("Source"))
    tot_i = sum(int(d[ie]) for d in data)
    tot_s = sum(int(d[st]) for d in data)
    print(f"launch {idx}: {s['name'][:70]}  warp-instr {tot_i}  stall samples {tot_s}")
    for i, d in sorted(sorted(enumerate(data), key=lambda x: -int(x[1][st]))[:top]):
        print(f"{i:5d} {d[src].strip()[:64]:64s} inst {int(d[ie]):>11d} stall {int(d[st]):>7d}")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--sass", type=int, default=None)
    ap.add_argument("--top", type=int, default=30)
    a = ap.parse_args()
    for i, r in enumerate(raw(a.report)):
        print(i, r["name"])
        print("   " + "  ".join(f"{k.split('.')[0].replace('__', ':')}={v[0]}{v[1]}" for k, v in r.items() if k != "name"))
    if a.sass is not None:
        sass(a.report, a.sass, a.top)
