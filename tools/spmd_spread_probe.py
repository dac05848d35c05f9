import json, sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2106_03219_b200 import runtime
dev = torch.device("cuda", 0)
x = runtime.synthetic(1 << 30, "f64", 0x210603219, device=dev)
for _ in range(20):
    runtime.reduce(x, sched="distribute", teams=148, threads=384)
for rep in range(4):
    with runtime.Trace(dev) as tr:
        runtime.reduce(x, sched="distribute", teams=148, threads=384)
    r = tr.records
    t0 = int(r["t_begin"][r["t_begin"] > 0].min())
    teams = r[r["kind"] == 1]
    comb = r[r["kind"] == 2][0]
    end = (teams["t_end"].astype(np.int64) - t0) / 1e3
    beg = (teams["t_begin"].astype(np.int64) - t0) / 1e3
    print(json.dumps({"rep": rep, "start_spread_us": round(float(beg.max() - beg.min()), 2),
        "first_end": round(float(end.min()), 1), "p10": round(float(np.percentile(end, 10)), 1),
        "p50": round(float(np.median(end)), 1), "p90": round(float(np.percentile(end, 90)), 1),
        "last_end": round(float(end.max()), 1), "mean_end": round(float(end.mean()), 1),
        "combine_us": round((int(comb["t_end"]) - int(comb["t_begin"])) / 1e3, 2),
        "span": round((int(comb["t_end"]) - t0) / 1e3, 1),
        "slowest_sms": [int(s) for s in teams["smid"][np.argsort(end)[-6:]]],
        "fastest_sms": [int(s) for s in teams["smid"][np.argsort(end)[:6]]]}), flush=True)
