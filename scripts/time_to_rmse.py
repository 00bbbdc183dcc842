"""Time to serial SGD's test RMSE (development tool; reads trace_compare.py output).

For each schedule of a trace file and target epochs e of the deterministic schedule's trace (exact
serial SGD, D-3), the first epoch at which the schedule's test RMSE is within 0.5% of serial
SGD's RMSE after e epochs, and the kernel time it took to get there.

python scripts/time_to_rmse.py profiles/r02ae_c2_f16.jsonl [--targets 1,2,5,10,20]
"""
import argparse
import json


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("trace")
    ap.add_argument("--targets", default="1,2,3,5,10,20")
    ap.add_argument("--tol", type=float, default=0.005)
    a = ap.parse_args()
    runs = [json.loads(line) for line in open(a.trace) if line.strip()]
    ser = next(r for r in runs if r["schedule"] == "deterministic")
    targets = [int(t) for t in a.targets.split(",") if int(t) <= len(ser["rmse"])]
    out = []
    for r in runs:
        row = {"cfg": r["cfg"], "storage": r["storage"], "schedule": r["schedule"],
               "ms_per_epoch": round(1e3 * sum(r["kernel_s"]) / len(r["kernel_s"]), 2), "reach": {}}
        for e in targets:
            goal = ser["rmse"][e - 1] * (1 + a.tol)
            hit = next((i for i, x in enumerate(r["rmse"]) if x <= goal), None)
            row["reach"][e] = None if hit is None else {
                "epochs": hit + 1, "ms": round(1e3 * sum(r["kernel_s"][:hit + 1]), 1)}
        out.append(row)
        print(json.dumps(row))


if __name__ == "__main__":
    main()
