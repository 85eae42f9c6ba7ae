"""profiles/<tag>_traffic.json from the per-kernel `--set full` raw CSVs of scripts/profile_round.sh:
DRAM bytes read + written, duration and tensor-pipe activity of one launch per kernel (developer tool).
usage: python scripts/traffic_from_ncu.py gpurun_out/prof_<tag> profiles/<tag>_traffic.json"""
import csv
import glob
import json
import os
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}


def main(src, dst):
    out = {}
    for f in sorted(glob.glob(os.path.join(src, "*_raw.csv"))):
        k = os.path.basename(f)[:-len("_raw.csv")]
        rows = list(csv.reader(open(f)))
        if len(rows) < 3:
            continue
        hdr, units, val = rows[0], rows[1], rows[2]

        def get(name):
            i = hdr.index(name)
            return float(val[i].replace(",", "")) * UNIT.get(units[i], 1.0)
        rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
        tp = [h for h in hdr if h.startswith("sm__pipe_tensor") and h.endswith("pct_of_peak_sustained_active")]
        out[k] = {"bytes": int(rd + wr), "read": int(rd), "write": int(wr),
                  "time_us": get("gpu__time_duration.sum"),
                  "tensor_active_pct": float(val[hdr.index(tp[0])]) if tp else None}
    json.dump(out, open(dst, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
