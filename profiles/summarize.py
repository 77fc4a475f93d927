"""Summarise ncu reports into small text files kept under profiles/ (the .ncu-rep files
stay in gpurun_out/, which is scratch).

    python profiles/summarize.py gpurun_out/prof_m32f.ncu-rep profiles/r01_m32_tma.txt "note" [launch]
"""

import collections
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__bytes_read.sum.per_second",
    "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__cycles_elapsed.avg.per_second",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "lts__t_sector_hit_rate.pct",
]


def ncu(rep, page, extra=()):
    r = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra], capture_output=True,
                       text=True)
    return list(csv.reader(io.StringIO(r.stdout)))


def main(rep, out, note="", launch=0):
    raw = ncu(rep, "raw")
    h, u, v = raw[0], raw[1], raw[2 + launch]
    lines = [f"# ncu summary of {rep.split('/')[-1]}", f"# {note}", ""]
    name_i = h.index("Kernel Name") if "Kernel Name" in h else None
    if name_i is not None:
        lines.append(f"kernel: {v[name_i]}")
    for k in KEYS:
        if k in h:
            i = h.index(k)
            lines.append(f"{k} = {v[i]} {u[i]}")
    src = ncu(rep, "source", ["--print-source", "sass", "--launch-skip", str(launch),
                              "--launch-count", "1"])
    if len(src) > 2:
        hdr = src[1]
        idx = {x: i for i, x in enumerate(hdr)}
        data = src[2:]
        cnt = collections.Counter()
        data = [r for r in data
                if len(r) >= len(hdr) and (r[idx["Instructions Executed"]] or "0").isdigit()]
        # ncu may print a kernel's SASS listing more than once (one section per source
        # view); every address counts once
        seen, uniq = set(), []
        for r in data:
            if r[idx["Address"]] not in seen:
                seen.add(r[idx["Address"]])
                uniq.append(r)
        data = uniq
        for r in data:
            toks = r[idx["Source"]].strip().split()
            if not toks:
                continue
            op = toks[1] if toks[0].startswith("@") else toks[0]
            cnt[op.split(".")[0]] += int(r[idx["Instructions Executed"]] or 0)
        tot = sum(cnt.values())
        lines += ["", f"executed warp-instructions: {tot}", "by opcode (share):"]
        for op, c in cnt.most_common(14):
            lines.append(f"  {op:10s} {c:12d}  {100.0 * c / max(tot, 1):5.1f}%")
        k = "Warp Stall Sampling (All Samples)"
        if k in idx:
            tot_s = sum(int(r[idx[k]] or 0) for r in data)
            lines += ["", f"top stall-sample sites (of {tot_s} samples):"]
            for r in sorted(data, key=lambda r: -int(r[idx[k]] or 0))[:8]:
                lines.append(f"  {r[idx[k]]:>6}  {r[idx['Source']].strip()[:90]}")
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "",
         int(sys.argv[4]) if len(sys.argv) > 4 else 0)
