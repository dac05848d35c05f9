"""Team timeline of config 4 (generic mode, 1024 teams x (32+256), 2^26):
int64 SPMD and fp64 ORDERED (where the last team folds the 1024 team partials
in team order after every team has finished).

    python tools/trace_generic.py [i64|f64] [spmd|ordered]"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2106_03219_b200 import runtime  # noqa: E402

dev = torch.device("cuda", 0)
dt = sys.argv[1] if len(sys.argv) > 1 else "i64"
ordered = len(sys.argv) > 2 and sys.argv[2] == "ordered"
x = runtime.synthetic(1 << 26, dt, 0x210603219, 4, device=dev)
o = torch.zeros(1, dtype=x.dtype, device=dev)
for _ in range(20):
    runtime.generic_reduce(x, teams=1024, par_threads=256, ordered=ordered, out=o)
with runtime.Trace(dev) as tr:
    runtime.generic_reduce(x, teams=1024, par_threads=256, ordered=ordered, out=o)
r = tr.records
teams = r[r["kind"] == 1]
comb = r[r["kind"] == 2]
t0 = int(teams["t_begin"].min())
beg = (teams["t_begin"].astype(np.int64) - t0) / 1e3
end = (teams["t_end"].astype(np.int64) - t0) / 1e3
dur = end - beg
print(json.dumps({
    "dtype": dt, "ordered": ordered, "teams": int(len(teams)), "sms": int(len(set(teams["smid"]))),
    "start_spread_us": round(float(beg.max()), 2),
    "team_duration_us_p50": round(float(np.median(dur)), 1),
    "team_duration_us_max": round(float(dur.max()), 1),
    "first_end_us": round(float(end.min()), 1), "last_end_us": round(float(end.max()), 1),
    "combine_end_us": round((int(comb["t_end"][0]) - t0) / 1e3, 1) if len(comb) else None,
    "combine_us": round((int(comb["t_end"][0]) - int(comb["t_begin"][0])) / 1e3, 2)
    if len(comb) else None,
    "end_p50_us": round(float(np.median(end)), 1),
    "ends_after_half": int((end > end.max() / 2).sum()),
    "teams_per_sm_max": int(np.bincount(teams["smid"]).max())}))
