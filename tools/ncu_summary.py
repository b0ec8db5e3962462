"""Summarise an ncu --set full report (kernel launches) into the numbers the
roofline uses: duration, DRAM bytes, L2 traffic, occupancy, stall mix.
usage: python tools/ncu_summary.py report.ncu-rep updates_per_launch [label]"""
import csv, io, json, subprocess, sys

rep = sys.argv[1]
upd = float(sys.argv[2])
label = sys.argv[3] if len(sys.argv) > 3 else rep
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}


def val(r, k):
    try:
        return float(r[ix[k]].replace(",", ""))
    except (KeyError, ValueError):
        return None


scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}
out = {"report": rep, "label": label, "launches": []}
for r in data:
    name = r[ix["Kernel Name"]] if "Kernel Name" in ix else "?"
    ms = val(r, "gpu__time_duration.sum")
    if units[ix["gpu__time_duration.sum"]] == "us":
        ms = ms / 1e3
    rd = val(r, "dram__bytes_read.sum")
    wr = val(r, "dram__bytes_write.sum")
    if rd is None:
        continue
    rd *= scale.get(units[ix["dram__bytes_read.sum"]], 1.0)
    wr *= scale.get(units[ix["dram__bytes_write.sum"]], 1.0)
    stalls = {h.replace("smsp__pcsamp_warps_issue_stalled_", ""): val(r, h) for h in hdr
              if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")}
    tot = sum(v for v in stalls.values() if v) or 1.0
    top = sorted(((k, v / tot) for k, v in stalls.items() if v), key=lambda x: -x[1])[:5]
    out["launches"].append({
        "kernel": name.split("(")[0], "ms": ms,
        "dram_read_GB": rd / 1e9, "dram_write_GB": wr / 1e9,
        "dram_bytes_per_update": (rd + wr) / upd,
        "dram_GBps": (rd + wr) / (ms / 1e3) / 1e9,
        "updates_per_s": upd / (ms / 1e3),
        "l2_hit_pct": val(r, "lts__t_sector_hit_rate.pct"),
        "l1_hit_pct": val(r, "l1tex__t_sector_hit_rate.pct"),
        # sector efficiency: useful bytes per 32-byte sector the LSU requested
        "ld_bytes_per_sector": val(r, "smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.ratio"),
        "st_bytes_per_sector": val(r, "smsp__sass_average_data_bytes_per_sector_mem_global_op_st.ratio"),
        "ldgsts_sectors_per_update": (val(r, "sm__sass_l1tex_t_sectors_pipe_lsu_mem_global_op_ldgsts_cache_bypass.sum")
                                      or 0) / upd,
        "ld_sectors_per_update": (val(r, "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum") or 0) / upd,
        "st_sectors_per_update": (val(r, "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum") or 0) / upd,
        "l2_throughput_pct": val(r, "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
        "dram_throughput_pct": val(r, "dram__throughput.avg.pct_of_peak_sustained_elapsed"),
        "sm_throughput_pct": val(r, "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
        "warps_active_per_sm": val(r, "sm__warps_active.avg.per_cycle_active"),
        "registers": val(r, "launch__registers_per_thread"),
        "l2_fabric_sectors_per_update": (val(r, "lts__t_sectors_srcunit_ltcfabric.sum") or 0) / upd,
        "top_stalls": top,
    })
print(json.dumps(out, indent=1))
