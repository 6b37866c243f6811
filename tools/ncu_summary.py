"""Summarise an `ncu --set full -k regex:exec_tile_kernel -c 8` capture of bench.py (one
launch per scheme, in SCHEMES order) into a markdown table, and record the mean DRAM bytes
per launch in profiles/ncu_traffic.json under the bench config key (the `traffic` field of
the bench line's roofline).

  python tools/ncu_summary.py REPORT.ncu-rep OUT.md --config "<bench config_key>" [--title T]
"""
import argparse
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCHEMES = ["tpl_nw", "tpl_wd", "to", "mvcc", "silo", "tictoc", "gputx", "gacco"]
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "smsp__warps_eligible.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
           "lts__t_requests_srcunit_tex.sum", "l1tex__m_l1tex2xbar_write_sectors_mem_global_op_atom.sum",
           "l1tex__m_l1tex2xbar_write_sectors_mem_global_op_red.sum",
           "smsp__thread_inst_executed_per_inst_executed.ratio"]
STALLS = "smsp__pcsamp_warps_issue_stalled_"


def raw(rep):
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True)
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return hdr, units, rows[2:]


def num(x):
    try:
        return float(x.replace(",", ""))
    except (ValueError, AttributeError):
        return 0.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("out")
    ap.add_argument("--config", required=True)
    ap.add_argument("--title", default="exec_tile_kernel, YCSB configs[1], tile 16")
    a = ap.parse_args()
    hdr, units, rows = raw(a.report)
    col = {h: i for i, h in enumerate(hdr)}
    dram_unit = units[col["dram__bytes_read.sum"]]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(dram_unit, 1e6)
    lines = [f"# ncu --set full: {a.title}", "",
             f"Report `{os.path.basename(a.report)}`; bench config `{a.config}`.",
             "Serialised, cold-cache replay (ncu flushes caches between passes): absolute times are not bench "
             "times; shares and traffic are what to read.", "",
             "| scheme | ms | DRAM MB | DRAM B/op | L2 hit % | L2 atom+red sectors (M/s) | threads/inst | warps active % | eligible/cycle | issue % | L1 % | L2 % | top stalls |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    per = []
    for s, r in zip(SCHEMES, rows):
        g = lambda m: num(r[col[m]]) if m in col else 0.0  # noqa: E731
        dram = (g("dram__bytes_read.sum") + g("dram__bytes_write.sum")) * scale
        per.append(dram)
        st = {h[len(STALLS):]: num(r[i]) for h, i in col.items()
              if h.startswith(STALLS) and not h.endswith("not_issued")}
        tot = sum(st.values()) or 1.0
        top = ", ".join(f"{k} {v / tot * 100:.0f}%" for k, v in sorted(st.items(), key=lambda t: -t[1])[:3])
        t_ms = g('gpu__time_duration.sum')
        tu = units[col["gpu__time_duration.sum"]]
        t_s = t_ms * {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1.0, "s": 1.0}.get(tu, 1e-3)
        atom = (g("l1tex__m_l1tex2xbar_write_sectors_mem_global_op_atom.sum")
                + g("l1tex__m_l1tex2xbar_write_sectors_mem_global_op_red.sum"))   # sectors sent to L2
        lines.append(f"| {s} | {t_s * 1e3:.3f} | {dram / 1e6:.0f} | {dram / (65536 * 16):.0f} | "
                     f"{g('lts__t_sector_hit_rate.pct'):.1f} | {atom / t_s / 1e6 if t_s else 0:.0f} | "
                     f"{g('smsp__thread_inst_executed_per_inst_executed.ratio'):.1f} | "
                     f"{g('sm__warps_active.avg.pct_of_peak_sustained_active'):.1f} | "
                     f"{g('smsp__warps_eligible.avg.per_cycle_active'):.3f} | "
                     f"{g('smsp__issue_active.avg.pct_of_peak_sustained_active'):.1f} | "
                     f"{g('l1tex__throughput.avg.pct_of_peak_sustained_active'):.1f} | "
                     f"{g('lts__throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | {top} |")
    mean = sum(per) / max(1, len(per))
    lines += ["", f"Mean DRAM bytes per launch: {mean / 1e6:.1f} MB over {len(per)} launches."]
    open(a.out, "w").write("\n".join(lines) + "\n")
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        entries = json.load(open(path))
    except Exception:
        entries = []
    entries = [e for e in entries if e.get("config") != a.config]
    entries.append({"config": a.config, "kernel": "exec_tile_kernel<*,YcsbWL,%s> (8 schemes, mean)" % (a.config.split("lanes=")[1].split()[0] if "lanes=" in a.config else "?"),
                    "dram_bytes_per_launch": mean, "source": os.path.relpath(a.out, ROOT)})
    json.dump(entries, open(path, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
