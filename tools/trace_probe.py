"""Team timeline of the bench construct from the device trace ring: when the
148 teams start and reach the last-team-finishes ticket, and how long the
ordered combine takes (fp64 sum, 2^30, distribute, 148x256; and ORDERED)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2106_03219_b200 import runtime  # noqa: E402

dev = torch.device("cuda", 0)
x = runtime.synthetic(1 << 30, "f64", 0x210603219, device=dev)
for _ in range(5):
    runtime.reduce(x, sched="distribute", teams=148, threads=256)
for mode in ("spmd", "ordered"):
    with runtime.Trace(dev) as tr:
        runtime.reduce(x, sched="distribute", teams=148, threads=256, mode=mode)
    r = tr.records
    t0 = int(r["t_begin"][r["t_begin"] > 0].min())
    if mode == "spmd":
        teams = r[r["kind"] == 1]
        comb = r[r["kind"] == 2][0]
        end = (teams["t_end"].astype(np.int64) - t0) / 1e3
        beg = (teams["t_begin"].astype(np.int64) - t0) / 1e3
        rec = {"mode": mode, "teams": int(len(teams)), "distinct_sms": int(len(set(teams["smid"]))),
               "start_spread_us": round(float(beg.max() - beg.min()), 2),
               "first_team_end_us": round(float(end.min()), 1),
               "last_team_end_us": round(float(end.max()), 1),
               "end_spread_us": round(float(end.max() - end.min()), 1),
               "end_p50_us": round(float(np.median(end)), 1),
               "combine_us": round((int(comb["t_end"]) - int(comb["t_begin"])) / 1e3, 2),
               "kernel_span_us": round((int(comb["t_end"]) - t0) / 1e3, 1)}
    else:
        st = r[r["kind"] == 3]
        fold = r[r["kind"] == 4][0]
        end = (st["t_end"].astype(np.int64) - t0) / 1e3
        rec = {"mode": mode, "stream_warps": int(len(st)),
               "streams_done_first_us": round(float(end.min()), 1),
               "streams_done_last_us": round(float(end.max()), 1),
               "folder_done_us": round((int(fold["t_end"]) - t0) / 1e3, 1),
               "folder_tail_us": round((int(fold["t_end"]) - int(st["t_end"].max())) / 1e3, 1)}
    print(json.dumps(rec), flush=True)

# where the ORDERED stream spread comes from: within an SM or across SMs
with runtime.Trace(dev) as tr:
    runtime.reduce(x, sched="distribute", teams=148, threads=256, mode="ordered")
r = tr.records
st = r[r["kind"] == 3]
t0 = int(r["t_begin"][r["t_begin"] > 0].min())
end = (st["t_end"].astype(np.int64) - t0) / 1e3
by_sm = {}
for s, e in zip(st["smid"].tolist(), end.tolist()):
    by_sm.setdefault(s, []).append(e)
within = [max(v) - min(v) for v in by_sm.values()]
means = [sum(v) / len(v) for v in by_sm.values()]
print(json.dumps({"ordered_stream_spread": {
    "within_sm_spread_us_mean": round(float(np.mean(within)), 1),
    "within_sm_spread_us_max": round(float(np.max(within)), 1),
    "across_sm_mean_end_spread_us": round(float(max(means) - min(means)), 1),
    "warps_per_sm": round(len(st) / len(by_sm), 1)}}), flush=True)
