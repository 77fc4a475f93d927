"""Per-KiB executed-instruction breakdown of one launch in an ncu report (reads the
source page; needs -lineinfo builds).

    python tools/ncu_ops.py gpurun_out/prof.ncu-rep [launch_index] [bytes_scanned]
"""

import collections
import csv
import io
import subprocess
import sys


def main(rep, skip=0, nbytes=1 << 30):
    r = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                        "--launch-skip", str(skip), "--launch-count", "1"],
                       capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(r)))
    name = rows[0][1] if rows and len(rows[0]) > 1 else "?"
    hdr = rows[1]
    idx = {x: i for i, x in enumerate(hdr)}
    cnt = collections.Counter()
    stall = collections.Counter()
    for row in rows[2:]:
        if len(row) < len(hdr):
            break  # next kernel section
        toks = row[idx["Source"]].strip().split()
        if not toks:
            continue
        op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
        cnt[op] += int(row[idx["Instructions Executed"]] or 0)
        stall[op] += int(row[idx["Warp Stall Sampling (All Samples)"]] or 0)
    kib = nbytes / 1024
    tot = sum(cnt.values())
    print(f"{name}: {tot / kib:.1f} warp-instructions per KiB")
    print("  " + "  ".join(f"{o}:{c / kib:.1f}" for o, c in cnt.most_common(24)))
    st = sum(stall.values()) or 1
    print("  stall samples by opcode: " +
          "  ".join(f"{o}:{100 * c / st:.0f}%" for o, c in stall.most_common(10)))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0,
         int(sys.argv[3]) if len(sys.argv) > 3 else 1 << 30)
