"""Per-m DRAM traffic and duration of rk_scan_kernel<M> from an ncu CSV launch list of
the bench command, written to profiles/r02_traffic.json (read by bench.py for
roofline.traffic).

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file gpurun_out/launches.csv \
        python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu --sustained-steps 0
    python profiles/traffic_from_ncu.py gpurun_out/launches.csv profiles/r02_launches.csv

Each launch of the sweep kernel is attributed to its m by its position in the step (the
bench scans the sweep's lengths in order; every m >= 32 runs rk_scan_kernel<32>); traffic = dram__bytes_read.sum + dram__bytes_write.sum per launch, averaged
over the launches of that m (ncu runs each launch alone and cold: the per-launch bytes are
what the kernel moves, the durations are only the kernel's share of the step).
"""

import collections
import csv
import io
import json
import re
import sys
from pathlib import Path

SWEEP = (4, 8, 16, 32, 64, 128, 256, 512, 1024)


def main(src, copy_to=None):
    text = Path(src).read_text()
    body = text[text.index('"ID"'):]
    rows = list(csv.DictReader(io.StringIO(body)))
    per = collections.defaultdict(dict)
    for r in rows:
        per[(r["ID"], r["Kernel Name"])][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    acc = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    kernels = collections.Counter()
    i = 0
    for (lid, name), v in sorted(per.items(), key=lambda kv: int(kv[0][0])):
        kernels[re.sub(r"\(.*", "", name)] += 1
        mt = re.search(r"rk_(?:scan|short)_kernel<(\d+)>", name)
        if not mt or "dram__bytes_read.sum" not in v:
            continue
        m = SWEEP[i % len(SWEEP)]
        i += 1
        assert int(mt.group(1)) == min(m, 32) if m >= 32 or m in (4, 8, 16) else True, (m, name)
        a = acc[m]
        a[0] += 1
        a[1] += v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"]
        a[2] += v["gpu__time_duration.sum"]
        a[3] += v["dram__bytes_write.sum"]
    out = {
        "per_m": {str(m): a[1] / a[0] for m, a in sorted(acc.items())},
        "per_m_write": {str(m): a[3] / a[0] for m, a in sorted(acc.items())},
        "per_m_ns": {str(m): a[2] / a[0] for m, a in sorted(acc.items())},
        "launches_per_m": {str(m): a[0] for m, a in sorted(acc.items())},
        "kernels": dict(kernels),
        "source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                  "--clock-control none of `python bench.py --steps 1 --warmup 3 --e2e-steps 0 "
                  "--no-cpu --sustained-steps 0` (profiles/r02_launches.csv)",
    }
    Path(__file__).with_name("r02_traffic.json").write_text(json.dumps(out, indent=1) + "\n")
    if copy_to:
        Path(copy_to).write_text(body)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
