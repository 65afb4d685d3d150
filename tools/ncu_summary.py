"""Summarise one `ncu --set full` capture of the step kernel (exported by
tools/capture_profiles.sh) into profiles/step_kernel_ncu.json, the file bench.py
reads for roofline.traffic and issue_roofline.

    python tools/ncu_summary.py PROF_DIR KERNEL_ID FISH SOURCE_NOTE > profiles/step_kernel_ncu.json
"""
import collections
import csv
import json
import os
import re
import sys

d, kernel_id, fish, note = sys.argv[1], sys.argv[2], int(float(sys.argv[3])), sys.argv[4]
raw = list(csv.reader(open(os.path.join(d, "step_raw.csv"))))
R = dict(zip(raw[0], raw[2]))
U = dict(zip(raw[0], raw[1]))


def num(key):
    v = float(R[key].replace(",", ""))
    u = U.get(key, "")
    return v * {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1.0, "usecond": 1.0, "msecond": 1e3,
                "nsecond": 1e-3}.get(u, 1.0)


rows = list(csv.reader(open(os.path.join(d, "step_source.csv"))))
hdr = rows[1]
i_src, i_exec = hdr.index("Source"), hdr.index("Thread Instructions Executed")
mix = collections.Counter()
for r in rows[2:]:
    if len(r) <= i_exec:
        continue
    m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[i_src])
    if m:
        mix[m.group(2)] += float(r[i_exec].replace(",", "") or 0)
tot = sum(mix.values())
top = dict((k, round(v / fish, 1)) for k, v in mix.most_common(12))
top["other"] = round((tot - sum(v for _, v in mix.most_common(12))) / fish, 1)
rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
out = {
    "source": note,
    "kernel_id": kernel_id,
    "kernel": R.get("Kernel Name", kernel_id),
    "fish": fish,
    "gpu__time_duration_us": num("gpu__time_duration.sum"),
    "dram_bytes_read_per_launch": rd,
    "dram_bytes_write_per_launch": wr,
    "dram_bytes_per_launch": rd + wr,
    "algorithmic_bytes_per_launch_80B": 80.0 * fish,
    "moved_bytes_per_launch_64B": 64.0 * fish,
    "warp_instructions_per_launch": num("smsp__inst_executed.sum"),
    "thread_instructions_per_fish": round(tot / fish, 1),
    "issue_active_pct": round(num("smsp__issue_active.avg.pct_of_peak_sustained_active"), 2),
    "warps_active_pct": round(num("sm__warps_active.avg.pct_of_peak_sustained_active"), 2),
    "fp64_pipe_active_pct": round(num("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"), 2),
    "alu_pipe_active_pct": round(num("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"), 2),
    "registers_per_thread": num("launch__registers_per_thread"),
    "grid": num("launch__grid_size"),
    "sm_clock_ghz": round(num("sm__cycles_elapsed.avg.per_second"), 4),
    "l2_hit_rate_pct": round(num("lts__t_sector_hit_rate.pct"), 2),
    "stalls_per_issue": {k.split("stalled_")[1].split("_per_issue")[0]: round(float(R[k]), 2)
                         for k in R if k.startswith("smsp__average_warps_issue_stalled_")
                         and float(R[k] or 0) >= 0.05},
    "note": "ncu flushes caches between replays (cold L2): DRAM bytes exclude the cross-step L2 reuse the "
            "bench sees; writes still in L2 at kernel end are not counted",
    "instruction_mix_per_fish": top,
}
print(json.dumps(out, indent=1))
