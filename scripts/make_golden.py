"""Write oracle golden traces (test RMSE per epoch) for full-size parity configs.

Calls only oracle/ (and the shared input generator datagen/).  Output:
tests/golden/<cfg>_<storage>_trace.json.  Usage:
    python scripts/make_golden.py C2 f32 [epochs] [shuffle_seed] [k]
The serial oracle runs at ~0.76 M updates/s (fp32) on one core, so C2 (99M samples) takes ~2 min
per epoch; run it in the background on the dev container.  fp16 epochs use the -mf16c build of the
oracle (ORACLE_F16C=1, bit-identical to the plain build: tests/test_oracle.py).  A k other than the
config's is written as <cfg>-k<K>_<storage>_trace.json.  The file is written as .partial after every
epoch and renamed when the run completes.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

os.environ.setdefault("ORACLE_F16C", "1")
import datagen  # noqa: E402
import oracle  # noqa: E402


def main():
    name, storage = sys.argv[1], sys.argv[2]
    cfg = datagen.CONFIGS[name]
    epochs = int(sys.argv[3]) if len(sys.argv) > 3 else cfg.epochs
    seed_sh = int(sys.argv[4]) if len(sys.argv) > 4 else cfg.seed_shuffle  # other seeds: the order's spread
    if len(sys.argv) > 5 and int(sys.argv[5]) != cfg.k:
        cfg = cfg.scaled(k=int(sys.argv[5]), name=f"{name}-k{sys.argv[5]}")
        name = cfg.name
    st = oracle.STORAGE_NAME[storage]
    (u, v, r), test = datagen.make(cfg)
    order = oracle.shuffle_perm(seed_sh, len(u))
    m = oracle.Model(cfg.m, cfg.n, cfg.k, st, seed=cfg.seed_init)
    tag = "" if seed_sh == cfg.seed_shuffle else f"_seed{seed_sh}"
    out = os.path.join(ROOT, "tests", "golden", f"{name}_{storage}{tag}_trace.json")
    rec = {"what": f"oracle test RMSE per epoch, serial SGD on the A-8 shuffled order (seed {seed_sh}), "
                   f"init A-7 (seed {cfg.seed_init}), {storage} storage",
           "written_by": "scripts/make_golden.py (calls only oracle/ and datagen/)",
           "config": cfg.__dict__, "rmse": [], "seconds": []}
    for t in range(epochs):
        t0 = time.time()
        rc = m.epoch(u, v, r, oracle.eta(cfg.alpha, cfg.beta, t), cfg.lam, order)
        assert rc == 0, "oracle diverged"
        rec["rmse"].append(m.rmse(*test))
        rec["seconds"].append(time.time() - t0)
        with open(out + ".partial", "w") as f:
            json.dump(rec, f, indent=1)
        print(t, rec["rmse"][-1], rec["seconds"][-1], flush=True)
    os.replace(out + ".partial", out)


if __name__ == "__main__":
    main()
