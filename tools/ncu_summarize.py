"""Turn gpurun_out/full_<cfg>.ncu-rep captures and launches_<cfg>.csv launch lists into the
tracked profiles/ artefacts:

  profiles/<tag>_ncu_full_<cfg>_f32_{raw,details}.csv   ncu -i ... --page raw|details --csv
  profiles/<tag>_launches_<cfg>_f32.csv                 the launch list, copied
  profiles/ncu_<cfg>_f32.json                           DRAM bytes / duration per kernel launch
                                                        (bench.py's roofline.traffic)

  python tools/ncu_summarize.py --tag r01_v3 [--configs c2 c3]
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import shutil
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def kname(full: str) -> str:
    """'void k_row_stats<float, 0>(Params)' -> 'k_row_stats'"""
    s = full.split("(")[0].split("<")[0]
    return s.split()[-1]


def raw_metrics(rep: str) -> list[dict]:
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True)
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    return [dict(zip(hdr, r)) for r in data], dict(zip(hdr, units)), out


SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def num(s: str) -> float:
    return float(s.replace(",", "")) if s not in ("", "n/a") else float("nan")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--configs", nargs="+", default=["c2", "c3"])
    ap.add_argument("--src", default=os.path.join(ROOT, "gpurun_out"))
    a = ap.parse_args()
    prof = os.path.join(ROOT, "profiles")
    for cfg in a.configs:
        rep = os.path.join(a.src, f"{a.tag}_full_{cfg}.ncu-rep")
        if not os.path.exists(rep):
            rep = os.path.join(a.src, f"full_{cfg}.ncu-rep")
        if os.path.exists(rep):
            recs, units, raw = raw_metrics(rep)
            with open(os.path.join(prof, f"{a.tag}_ncu_full_{cfg}_f32_raw.csv"), "w") as f:
                f.write(raw)
            det = subprocess.check_output(["ncu", "-i", rep, "--page", "details", "--csv"], text=True)
            with open(os.path.join(prof, f"{a.tag}_ncu_full_{cfg}_f32_details.csv"), "w") as f:
                f.write(det)
            summary = {"source": f"profiles/{a.tag}_ncu_full_{cfg}_f32_raw.csv (ncu --set full "
                                 "--clock-control none, one launch of each kernel, call 11)"}
            for r in recs:
                k = kname(r["Kernel Name"])
                rd = num(r["dram__bytes_read.sum"]) * SCALE[units["dram__bytes_read.sum"]]
                wr = num(r["dram__bytes_write.sum"]) * SCALE[units["dram__bytes_write.sum"]]
                assert units["gpu__time_duration.sum"] == "us"
                summary[f"{k}_dram_bytes_per_launch"] = rd + wr
                summary[f"{k}_duration_us_ncu"] = num(r["gpu__time_duration.sum"])
            with open(os.path.join(prof, f"ncu_{cfg}_f32.json"), "w") as f:
                json.dump(summary, f, indent=1)
            print(cfg, summary)
        lst = os.path.join(a.src, f"{a.tag}_launches_{cfg}.csv")
        if not os.path.exists(lst):
            lst = os.path.join(a.src, f"launches_{cfg}.csv")
        if os.path.exists(lst):
            shutil.copy(lst, os.path.join(prof, f"{a.tag}_launches_{cfg}_f32.csv"))
            share = defaultdict(float)
            with open(lst) as f:
                lines = [l for l in f if l.startswith('"')]
            for r in csv.DictReader(io.StringIO("".join(lines))):
                if r.get("Metric Name") == "gpu__time_duration.sum":
                    share[kname(r["Kernel Name"])] += num(r["Metric Value"])
            tot = sum(share.values())
            print(cfg, "launch-list share:", {k: round(v / tot, 3) for k, v in share.items()})


if __name__ == "__main__":
    main()
