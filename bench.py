"""Benchmark: SGD updates/s of the batch-Hogwild! epoch (PAPER.md:207 metric) on the Netflix-shaped
synthetic workload (BASELINE.json configs[1]), k = 128, on one B200; with --gpus N > 1 the partitioned
path on the Hugewiki-shaped workload split over the N GPUs (BASELINE.json configs[3], strong scaling).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--storage f16|f32|bf16] [--config C2] [--schedule hogwild|wavefront_cta|...]
                    [--scaling weak|strong]

One step = one epoch of the hot path over the whole training set (N = 99,072,112 updates) followed by
the test-RMSE evaluation, both in libmf.so's kernels.  Prints ONE JSON line (rank 0).
`value` is device-timed with inputs resident in HBM; `e2e` repeats the step through the public C ABI
from pinned HOST buffers (batch-Hogwild!: mf_epoch_host streams R from host memory every step, H2D
overlapped with the update kernel; other schedules: mf_load_coo H2D + validation + A-8 shuffle,
mf_epoch), then mf_rmse with the test set from host memory and the result D2H.
N > 1 (torchrun): the partitioned path with NCCL Q rotation, one process per GPU, max-over-ranks time
(defaults: --config C4 --scaling strong --storage f16).  N = 1 also runs, in `other_runs`, the other
storage, the CTA wavefront and deterministic schedules on the same workload, the Yahoo!Music shape
(batch-Hogwild!, both wavefront forms: configs[2]) and the Hugewiki shape on this one GPU (batch-Hogwild!,
CTA wavefront and the 1-partition partitioned path: configs[3]; --no-c4 skips it).
`--impl reference` times the CPU oracle (the only reference this paper-only task has) on a bounded
sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import datagen  # noqa: E402

HBM_FALLBACK_GBS = 6650.0  # B200_PROFILING.md fallback, used only if MEASURED_PEAKS.json is absent


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback"


def l2_peaks(row_bytes):
    """Measured L2 ceilings (scripts/l2_ceiling.cu on a B200, profiles/r02_l2_ceiling.jsonl): the best
    random-row read-modify-write bandwidth for rows of `row_bytes` resident in L2 (the update kernels'
    own L2 access shape) and the best contiguous read+write bandwidth; (None, None) if absent."""
    rows, stream = None, None
    try:
        with open(os.path.join(ROOT, "profiles", "r02_l2_ceiling.jsonl")) as f:
            for line in f:
                d = json.loads(line)
                if d.get("pattern") == "rows_rw" and d.get("row_bytes") == row_bytes:
                    rows = max(rows or 0.0, d["GBps"])
                elif d.get("pattern") == "stream_rw":
                    stream = max(stream or 0.0, d["GBps"])
    except Exception:
        pass
    return rows, stream


def cpu_info():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return model, os.cpu_count()


SHAPE_NAME = {"C1": "planted rank-8 parity config", "C2": "Netflix-shaped", "C3": "Yahoo!Music-shaped",
              "C4": "Hugewiki-shaped"}


def roofline(cfg, storage, N, k_s, traffic, schedule):
    """Roofline object of the update kernel, against the resource that binds it.

    L2: the algorithmic bytes B_alg = 12 + 4kb per update all pass through L2 (triple,
    p_u and q_v read, both rows written; the CTA wavefront keeps q_v on chip, so 12 + 2kb reach L2),
    against the L2's measured ceiling for random-row read-modify-write.  HBM: the DRAM bytes of one
    launch (ncu, when captured for this config) or, failing that, the compulsory 12 + 2kb (R stream + P
    rows; Q is L2-resident at every configured shape), against the measured HBM copy peak.  `bound` is
    the one of the two the kernel is closer to (the larger fraction); both are reported."""
    b = 4 if storage == "f32" else 2
    hbm, hbm_kind = peaks()
    on_chip_q = schedule == "wavefront_cta"
    B = b_alg(cfg.k, storage)
    B_l2 = 12 + 2 * cfg.k * b if on_chip_q else B
    l2_rows, l2_stream = l2_peaks(cfg.k * b)
    b_hbm = 12 + 2 * cfg.k * b
    dram = traffic / N if traffic else b_hbm
    l2 = None
    if l2_rows:
        l2 = {"achieved": B_l2 * N / k_s / 1e9, "peak": l2_rows, "unit": "GB/s",
              "peak_kind": "measured L2 random-row RMW ceiling, %d-B rows (scripts/l2_ceiling.cu, "
                           "profiles/r02_l2_ceiling.jsonl)" % (cfg.k * b),
              "bytes_per_update": B_l2, "stream_rw_peak": l2_stream}
        l2["frac"] = l2["achieved"] / l2["peak"]
    hb = {"achieved": dram * N / k_s / 1e9, "peak": hbm, "peak_kind": hbm_kind, "unit": "GB/s",
          "frac": dram * N / k_s / 1e9 / hbm, "bytes_per_update": dram,
          "basis": "ncu dram__bytes_read+write of one launch" if traffic else
                   "compulsory 12 + 2kb (R + P rows; Q L2-resident)",
          "frac_compulsory": b_hbm * N / k_s / 1e9 / hbm, "frac_alg_bytes": B * N / k_s / 1e9 / hbm}
    top = l2 if l2 and l2["frac"] >= hb["frac"] else hb
    roof = {"bound": "l2" if top is l2 else "hbm", "achieved": top["achieved"], "peak": top["peak"],
            "unit": "GB/s", "frac": top["frac"], "traffic": traffic, "peak_kind": top["peak_kind"],
            "bytes_per_update_alg": B, "updates_per_launch": N, "kernel_ms": k_s * 1e3,
            "l2": l2, "hbm": hb}
    return roof


def b_alg(k, storage):
    """algorithmic bytes per update = 12 (triple) + 2kb (read p, q) + 2kb (write p, q)."""
    b = 4 if storage == "f32" else 2
    return 12 + 4 * k * b


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        time.sleep(0.25)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        time.sleep(0.15)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for nm, val in zip(names, r[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        loaded = sorted(sm)[len(sm) // 2:] if sm else []
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def load_traffic(storage, cfgname, schedule="hogwild"):
    """ncu dram bytes per launch of the update kernel for this (config, storage, schedule), from the
    committed profile summary profiles/ncu_summary.json (or None)."""
    key = f"{cfgname}/{storage}" if schedule == "hogwild" else f"{cfgname}-wfcta/{storage}"
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            d = json.load(f)
        return d["kernels"][key]["dram_bytes_per_launch"]
    except Exception:
        return None


def load_pattern_ceiling(cfg, storage, p_only=False):
    """Best updates/s of scripts/sgd_mem_ceiling.cu (the update's exact row traffic -- triple stream,
    p_u and q_v read + written through L2 -- without its arithmetic) for this workload's shape, from the
    committed sweep profiles/r01c_mem_ceiling.jsonl (or None).  It is the memory system's ceiling for
    batch-Hogwild!'s access pattern: above the HBM roofline when Q is L2-resident."""
    row_bytes = cfg.k * (4 if storage == "f32" else 2)
    try:
        best, match = None, False
        name = "r01c_mem_ceiling_p_only.jsonl" if p_only else "r01c_mem_ceiling.jsonl"
        with open(os.path.join(ROOT, "profiles", name)) as f:
            for line in f:
                d = json.loads(line)
                if "m" in d:
                    match = (d["m"], d["n"], d["N"], d["row_bytes"]) == (cfg.m, cfg.n, cfg.n_train, row_bytes)
                elif match:
                    u = max(d["updates_per_s_D1"], d["updates_per_s_D2"])
                    best = u if best is None else max(best, u)
        return best
    except Exception:
        return None


# ----------------------------------------------------------------- reference
def run_reference(a, cfg):
    """The oracle as it stands (serial C++, 1 core) on a bounded sample of the same workload."""
    import oracle
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    st = oracle.STORAGE_NAME[a.storage]
    G = int(os.environ.get("WORLD_SIZE", "1"))
    # the same workload as our arm (for G > 1: rank 0's shard of the partitioned problem, with the
    # factors at full global size)
    if G == 1:
        (u, v, r), test = datagen.make(cfg)
        m_glob = cfg.m
    else:
        (u, v, r), test = shard(cfg, G, 0, a.scaling)
        m_glob = partition_shape(cfg, G, a.scaling)[0]
    m = oracle.Model(m_glob, cfg.n, cfg.k, st, seed=cfg.seed_init)
    eta = oracle.eta(cfg.alpha, cfg.beta, 0)
    # bound the run: size each step so warmup + steps take ~2 minutes on this core
    t0 = time.perf_counter()
    m.epoch(u[:50_000], v[:50_000], r[:50_000], eta, cfg.lam)
    speed = 50_000 / (time.perf_counter() - t0)
    sample = int(min(a.ref_sample, max(10_000, speed * 120.0 / (a.warmup + a.steps))))
    times = []
    for i in range(a.warmup + a.steps):
        lo = (i * sample) % max(1, len(u) - sample)
        t0 = time.perf_counter()
        m.epoch(u[lo:lo + sample], v[lo:lo + sample], r[lo:lo + sample], eta, cfg.lam)
        dt = time.perf_counter() - t0
        if i >= a.warmup:
            times.append(dt)
    tot = sum(times)
    val = a.steps * sample / tot
    desc = f"{sample} consecutive shuffled samples of {cfg.name} per step, full-size P/Q, {a.storage} storage"
    out = {"metric": "sgd_updates_per_sec", "value": val, "unit": "updates/s", "n_gpus": a.gpus,
           "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * tot / a.steps, "higher_is_better": True,
           "scaling": a.scaling, "vs_baseline": None, "dtype": "f32", "storage": a.storage, "data": "synthetic",
           "impl": "reference",
           "config": workload_config(cfg, G, a.storage, a.schedule if G == 1 else "partitioned", a.scaling),
           "arm": {"what": "serial C++ oracle (oracle/mf_oracle.cpp), 1 core", "sample_per_step": sample},
           "cpu_baseline": {"value": val, "unit": "updates/s", "cores": 1, "kind": "oracle", "sample": desc,
                            "cpu_model": cpu_info()[0], "host_cpus": cpu_info()[1]},
           "e2e": {"value": val, "unit": "updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def partition_shape(cfg, G, scaling):
    """(m_glob, rows per rank via mf_segment, train / test samples per rank) of the G-rank problem.
    weak: every rank owns a full cfg-shaped row segment (m_glob = G m, N = G n_train), per-GPU work
    fixed; strong: cfg itself is split into G row segments (C4 at 2/4/8 GPUs, BASELINE configs[3])."""
    if scaling == "strong":
        return cfg.m, cfg.n_train // G, cfg.n_test // G
    return cfg.m * G, cfg.n_train, cfg.n_test


def shard(cfg, G, rank, scaling):
    """Rank `rank`'s training / test shard: draws of ONE global planted model restricted to the rank's
    row segment (datagen.make_segment), so the G ranks factorise one consistent matrix."""
    m_glob, n_tr, n_te = partition_shape(cfg, G, scaling)
    pb, pe = rank * m_glob // G, (rank + 1) * m_glob // G  # mf_segment's balanced row segment (mf.h)
    return datagen.make_segment(cfg, m_glob, pb, pe, n_tr, n_te, rank)


def workload_config(cfg, G, storage, schedule, scaling="weak"):
    """The `config` object, identical for both arms of the same run."""
    b = 4 if storage == "f32" else 2
    if G == 1:
        return {"workload": f"{cfg.name}: {SHAPE_NAME.get(cfg.name, cfg.name)} (PAPER.md Table 2) m={cfg.m} "
                            f"n={cfg.n} N={cfg.n_train} k={cfg.k}, planted rank-8 synthetic ratings",
                "schedule": schedule, "storage": storage, "alpha": cfg.alpha, "beta": cfg.beta, "lambda": cfg.lam,
                "l2": "inputs larger than L2 (R %.2f GB, P %.0f MB); no flush" % (12 * cfg.n_train / 1e9,
                                                                                  cfg.m * cfg.k * b / 1e6),
                "step": "one epoch over all N ratings (mf_epoch) + test RMSE (mf_rmse)"}
    m_glob, n_tr, _ = partition_shape(cfg, G, scaling)
    what = ("one %s-shaped row segment per GPU (weak scaling)" % cfg.name if scaling == "weak" else
            "%s split into %d row segments (strong scaling)" % (cfg.name, G))
    return {"workload": f"{cfg.name} ({SHAPE_NAME.get(cfg.name, cfg.name)}) partitioned over {G} GPUs: m={m_glob} "
                        f"n={cfg.n} N={n_tr * G} k={cfg.k}, {what}; one global planted rank-8 model",
            "schedule": "partitioned (S passes x G rounds; unit grid of 2G half-segment Q units, each family "
                        "rotating by its own Latin square over NCCL send/recv, overlapped with the other's updates)",
            "storage": storage, "parallelism": f"P row segments x rotating Q segments over {G} GPUs",
            "alpha": cfg.alpha, "beta": cfg.beta, "lambda": cfg.lam, "l2": "inputs larger than L2; no flush",
            "step": "one epoch (mf_epoch partitioned) + test RMSE (mf_rmse, collective)"}


def cpu_baseline(cfg, storage, u, v, r, budget_s=12.0):
    """Oracle updates/s on a bounded sample (full-size factors), 1 core."""
    import oracle
    st = oracle.STORAGE_NAME[storage]
    m = oracle.Model(cfg.m, cfg.n, cfg.k, st, seed=cfg.seed_init)
    eta = oracle.eta(cfg.alpha, cfg.beta, 0)
    n, done, t_all = 100_000, 0, 0.0
    while t_all < budget_s and done + n <= len(u):
        t0 = time.perf_counter()
        m.epoch(u[done:done + n], v[done:done + n], r[done:done + n], eta, cfg.lam)
        t_all += time.perf_counter() - t0
        done += n
    model, nproc = cpu_info()
    return {"value": done / t_all, "unit": "updates/s", "cores": 1, "kind": "oracle", "cpu_model": model,
            "host_cpus": nproc,
            "sample": f"first {done} samples of {cfg.name} in stored order, full-size P/Q, {storage} storage, "
                      f"{t_all:.1f} s on 1 of {nproc} host CPUs ({model})"}


# ---------------------------------------------------------------------- ours
def resolve_defaults(a, world):
    """N = 1: BASELINE.json configs[1] (Netflix shape, batch-Hogwild!, fp16 storage).  N > 1 (or
    --partitioned): configs[3], the Hugewiki shape split over the N GPUs (strong scaling), fp16 storage."""
    multi = world > 1 or a.partitioned
    a.config = a.config or ("C4" if multi else "C2")
    a.scaling = a.scaling or ("strong" if multi else "weak")
    a.storage = a.storage or "f16"
    return a


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--storage", default=None, choices=["f16", "f32", "bf16"])
    ap.add_argument("--config", default=None, help="default C2 (one GPU), C4 (N > 1)")
    ap.add_argument("--schedule", default="hogwild",
                    choices=["hogwild", "wavefront", "wavefront_cta", "deterministic"])
    ap.add_argument("--workers", type=int, default=0)
    ap.add_argument("--variant", type=int, default=-1)
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-variants", action="store_true", help="skip the other storage / schedule runs")
    ap.add_argument("--partitioned", action="store_true",
                    help="run the multi-GPU (NCCL, partitioned) path even at one rank")
    ap.add_argument("--ref-sample", type=int, default=1_000_000)
    ap.add_argument("--scaling", default=None, choices=["weak", "strong"],
                    help="N > 1: strong (default) = --config split over N; weak = one --config-shaped row segment "
                         "per GPU")
    ap.add_argument("--no-c4", action="store_true", help="N = 1: skip the Hugewiki-shaped runs in other_runs")
    a = ap.parse_args()
    a.warmup = max(a.warmup, 3)
    resolve_defaults(a, int(os.environ.get("WORLD_SIZE", "1")))
    cfg = datagen.CONFIGS[a.config]

    if a.impl == "reference":
        return run_reference(a, cfg)

    import torch
    import torch.distributed as dist
    from paper_1610_05838_b200 import mf

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 or a.partitioned:
        return run_partitioned(a, cfg, rank, world, local)
    torch.cuda.set_device(local)
    stream = torch.cuda.current_stream()

    (u, v, r), (tu, tv, tr) = datagen.make(cfg)
    N = len(u)
    variant = a.variant if a.variant >= 0 else 0
    # inputs resident in HBM (torch tensors as device memory), loaded through the C ABI
    du, dv, dr = (torch.from_numpy(x).cuda() for x in (u, v, r))
    dtu, dtv, dtr = (torch.from_numpy(x).cuda() for x in (tu, tv, tr))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def measure(storage, schedule, steps, warmup, clk=None, **opts):
        """Device-timed steps (epoch + test RMSE) with inputs resident in HBM."""
        if schedule == "wavefront_cta":
            schedule, opts = "wavefront", dict(opts, wave_cta=1)
        var = a.variant if a.variant >= 0 else 0
        g = mf.MF(cfg.m, cfg.n, cfg.k, cfg.alpha, cfg.lam, cfg.seed_init, storage=storage, beta=cfg.beta,
                  seed_shuffle=cfg.seed_shuffle, device=local, stream=stream.cuda_stream, variant=var,
                  workers=a.workers, **opts)
        g.load(du, dv, dr)
        for _ in range(warmup):
            g.epoch(schedule)
            g.rmse(dtu, dtv, dtr)
        kern, launches, rm, workers = [], 0, None, 0
        torch.cuda.synchronize()
        if clk:
            clk.__enter__()
        e0.record(stream)
        for _ in range(steps):
            st = g.epoch(schedule)
            rm = g.rmse(dtu, dtv, dtr)
            kern.append(st.kernel_seconds)
            launches += st.launches + 3  # + validate, rmse, final-sum kernels of mf_rmse
            workers = st.workers
        e1.record(stream)
        torch.cuda.synchronize()
        if clk:
            clk.__exit__(None, None, None)
        var_eff = int(g.get(mf.MF_OPT_VARIANT))  # the auto fields resolved (hogwild L2 prefetch pick)
        kappa = g.get(mf.MF_OPT_Q_KAPPA)  # batch-Hogwild!: expected concurrent updates per Q row (A-20)
        g.close()
        ms_ = e0.elapsed_time(e1) / steps
        return {"ms": ms_, "value": N / (ms_ * 1e-3), "kernel_s": statistics.mean(kern), "launches": launches,
                "rmse": rm, "workers": workers, "epochs_done": warmup + steps, "variant": var_eff,
                "q_kappa": kappa if kappa >= 0 else None}

    clk = Clocks(local)
    head = measure(a.storage, a.schedule, a.steps, a.warmup, clk=clk)
    ms, value, launches, workers = head["ms"], head["value"], head["launches"], head["workers"]
    rmses = [head["rmse"]]

    # roofline of the dominant kernel (the update kernel): algorithmic bytes / its event-timed duration
    k_s = head["kernel_s"]
    traffic = load_traffic(a.storage, cfg.name, a.schedule)
    roof = roofline(cfg, a.storage, N, k_s, traffic, a.schedule)
    roof.update({"kernel": "k_hogwild" if a.schedule == "hogwild" else "k_" + a.schedule,
                 "kernel_share_of_step": k_s * 1e3 / ms})
    peak = roof["hbm"]["peak"]
    ceil = (load_pattern_ceiling(cfg, a.storage, p_only=(a.schedule == "wavefront_cta"))
            if a.schedule in ("hogwild", "wavefront_cta") else None)
    if ceil:
        roof["pattern_ceiling_updates_per_s"] = ceil
        roof["frac_of_pattern_ceiling"] = (N / k_s) / ceil
        roof["pattern_ceiling_source"] = "scripts/sgd_mem_ceiling.cu sweep, profiles/r01c_mem_ceiling.jsonl"

    # the other storage and the wavefront schedule (CTA workers, Q in shared memory), same workload
    others = {}
    if not a.no_variants:
        other_st = "f32" if a.storage != "f32" else "f16"
        for key, st_, sch, opts in ((f"hogwild/{other_st}", other_st, "hogwild", {}),
                                    (f"wavefront_cta/{a.storage}", a.storage, "wavefront", {"wave_cta": 1}),
                                    (f"wavefront_cta/{other_st}", other_st, "wavefront", {"wave_cta": 1}),
                                    (f"deterministic/{a.storage}", a.storage, "deterministic", {})):
            res = measure(st_, sch, max(3, a.steps // 5), 3, **opts)
            res["alg_GBps"] = b_alg(cfg.k, st_) * N / res["kernel_s"] / 1e9
            rf = roofline(cfg, st_, N, res["kernel_s"], load_traffic(st_, cfg.name, key.split("/")[0]),
                          key.split("/")[0])
            res["roofline_frac"] = rf["frac"]
            res["roofline_bound"] = rf["bound"]
            res["hbm_frac"] = rf["hbm"]["frac"]
            res["l2_frac"] = (rf["l2"] or {}).get("frac")
            # against the memory-pattern ceiling of the kernel's own global traffic (p+q rows for
            # batch-Hogwild!, p rows only for the CTA wavefront whose Q group is on chip)
            ceil = load_pattern_ceiling(cfg, st_, p_only=(sch == "wavefront")) if sch != "deterministic" else None
            res["frac_of_pattern_ceiling"] = (N / res["kernel_s"]) / ceil if ceil else None
            others[key] = {k_: res[k_] for k_ in ("value", "ms", "kernel_s", "rmse", "workers", "alg_GBps",
                                                  "roofline_bound", "roofline_frac", "hbm_frac", "l2_frac",
                                                  "epochs_done",
                                                  "variant", "frac_of_pattern_ceiling")}

    if not a.no_variants and a.config == "C2":
        others.update(c5_leg(mf, stream, local, cfg, (du, dv, dr), (dtu, dtv, dtr)))
        others.update(c3_leg(mf, stream, local, a.storage))
    if not a.no_variants and not a.no_c4 and a.config != "C4":
        others.update(c4_leg(mf, stream, local, a.storage))

    # end to end through the public API from pinned host buffers
    hu, hv, hr = (torch.from_numpy(x).pin_memory() for x in (u, v, r))
    htu, htv, htr = (torch.from_numpy(x).pin_memory() for x in (tu, tv, tr))
    sched = "wavefront" if a.schedule == "wavefront_cta" else a.schedule
    ge = mf.MF(cfg.m, cfg.n, cfg.k, cfg.alpha, cfg.lam, cfg.seed_init, storage=a.storage, beta=cfg.beta,
               seed_shuffle=cfg.seed_shuffle, device=local, stream=stream.cuda_stream, variant=variant,
               workers=a.workers, wave_cta=int(a.schedule == "wavefront_cta"))

    streamed = sched == "hogwild"

    def e2e_step():
        if streamed:
            # mf_epoch_host: R streamed from pinned host memory in chunks, H2D overlapped with the update
            # kernel; the synthetic draws are i.i.d., i.e. already in random order (A-8)
            ge.epoch_host(hu, hv, hr)
        else:
            ge.load(hu, hv, hr)      # H2D + device validation + A-8 shuffle
            ge.epoch(sched)
        return ge.rmse(htu, htv, htr)  # H2D of the test set, RMSE kernels, D2H of the result

    e2e_step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record(stream)
    for _ in range(a.e2e_steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / a.e2e_steps
    wall_ms = (time.perf_counter() - t0) * 1e3 / a.e2e_steps
    ge.close()
    h2d = 12 * N + 12 * len(tu)

    cpu = None if a.no_cpu else cpu_baseline(cfg, a.storage, u, v, r)
    out = {
        "metric": "sgd_updates_per_sec", "value": value, "unit": "updates/s", "n_gpus": 1, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32", "storage": a.storage, "data": "synthetic",
        "config": workload_config(cfg, 1, a.storage, a.schedule),
        "arm": {"workers": workers, "batch_f": 256, "variant": head["variant"],
                "l2_row_prefetch": ((head["variant"] >> 16) & 0xF) not in (0, 15),
                "q_kappa": head["q_kappa"],
                "q_write_back": None if head["q_kappa"] is None else
                ("atomic add" if head["q_kappa"] < 0.5 else "store") + " (MF_OPT_Q_UPDATE auto, DESIGN.md A-20)"},
        "test_rmse": rmses[-1],
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": {"value": N / (e2e_ms * 1e-3), "unit": "updates/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": 8, "ms_per_step": e2e_ms, "wall_ms_per_step": wall_ms,
                "includes": ("mf_epoch_host: every step streams R (12 B/sample) from pinned host memory in "
                             "2^22-sample chunks, device validation per chunk, batch-Hogwild! overlapped with "
                             "the copies; then mf_rmse with the test set copied from pinned host, result D2H"
                             if streamed else
                             "mf_load_coo (H2D of R from pinned host, validation, A-8 shuffle), mf_epoch, "
                             "mf_rmse (H2D of the test set), result D2H")},
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "test_rmse_epochs": head["epochs_done"],
        "other_runs": others,
    }
    print(json.dumps(out), flush=True)


def shape_leg(mf, stream, local, storage, name, schedules, epochs=5):
    """Another BASELINE.json workload on THIS one GPU, as extra lines of `other_runs`: C3 (configs[2], the
    Yahoo!Music shape, "wavefront-update vs batch-Hogwild!") and C4 (configs[3], the Hugewiki shape: N =
    3,069,817,980, m = 50M, n = 39,781 -- R 36.8 GB and P 12.8 GB fp16 resident, HBM binds since P is 100x
    the L2; the partitioned schedule with one partition runs the multi-GPU code path's kernels and
    launches).  Synthetic draws are i.i.d., so the stored order is already random (A-8, MF_OPT_SHUFFLE =
    0).  Epochs 0-2 of the auto-tuned schedules are their prefetch trials; the kernel time reported is the
    mean of the later epochs; the test RMSE after `epochs` epochs is reported beside it."""
    import gc
    cfg = datagen.CONFIGS[name]
    t0 = time.perf_counter()
    (u, v, r), (tu, tv, tr) = datagen.make(cfg)
    gen_s = time.perf_counter() - t0
    N = len(u)
    out = {}
    for label, sched, opts in schedules:
        g = mf.MF(cfg.m, cfg.n, cfg.k, cfg.alpha, cfg.lam, cfg.seed_init, storage=storage, beta=cfg.beta,
                  seed_shuffle=cfg.seed_shuffle, device=local, stream=stream.cuda_stream, shuffle=0, **opts)
        g.load(u, v, r)
        ks = []
        for _ in range(epochs):
            ks.append(g.epoch(sched).kernel_seconds)
        rm = g.rmse(tu, tv, tr)
        passes = int(g.get(mf.MF_OPT_WAVE_PASSES)) if sched == "wavefront" else None
        g.close()
        k_s = statistics.mean(ks[3:]) if sched != "partitioned" else statistics.mean(ks[1:])
        sname = "wavefront_cta" if opts.get("wave_cta") else "hogwild"
        rf = roofline(cfg, storage, N, k_s, load_traffic(storage, name, sname), sname)
        out[f"{name}:{label}/{storage}"] = {"value": N / k_s, "kernel_s": k_s, "rmse_after_%d_epochs" % epochs: rm,
                                            "roofline_bound": rf["bound"], "roofline_frac": rf["frac"],
                                            "hbm": rf["hbm"], "l2_frac": (rf["l2"] or {}).get("frac"), "N": N,
                                            **({"wave_passes": passes} if passes else {})}
    out[f"{name}:note"] = ("kernel-timed (CUDA events inside libmf), inputs resident; host generation %.0f s"
                           % gen_s)
    del u, v, r
    gc.collect()
    return out


def c4_leg(mf, stream, local, storage, epochs=5):
    return shape_leg(mf, stream, local, storage, "C4",
                     (("hogwild", "hogwild", {}), ("wavefront_cta", "wavefront", {"wave_cta": 1}),
                      ("partitioned_1", "partitioned", {"partitions": 1})), epochs)


def c5_leg(mf, stream, local, cfg, train, test, epochs=5):
    """BASELINE.json configs[4]: the k sweep on the Netflix shape (the headline's own inputs, resident), batch-
    Hogwild! in fp16 and fp32 storage, k = 32 / 64 / 256 (k = 128 is the headline and the `hogwild/f32`
    line).  Kernel time = mean of the epochs after the prefetch trials (epochs 0-2); roofline per k against
    the L2 ceiling (B_alg = 12 + 4kb) and, from the committed ncu bytes for that k, HBM."""
    N = len(train[0])
    out = {}
    for storage in ("f16", "f32"):
        for k in (32, 64, 256):
            kc = cfg.scaled(k=k)
            g = mf.MF(kc.m, kc.n, k, kc.alpha, kc.lam, kc.seed_init, storage=storage, beta=kc.beta,
                      seed_shuffle=kc.seed_shuffle, device=local, stream=stream.cuda_stream)
            g.load(*train)
            ks = [g.epoch("hogwild").kernel_seconds for _ in range(epochs)]
            rm = g.rmse(*test)
            g.close()
            k_s = statistics.mean(ks[3:])
            rf = roofline(kc, storage, N, k_s, load_traffic(storage, f"C2-k{k}"), "hogwild")
            row = {"value": N / k_s, "kernel_s": k_s, "rmse_after_%d_epochs" % epochs: rm,
                   "roofline_bound": rf["bound"], "roofline_frac": rf["frac"],
                   "l2_frac": (rf["l2"] or {}).get("frac"), "hbm_frac": (rf["hbm"] or {}).get("frac"),
                   "alg_GBps": b_alg(k, storage) * N / k_s / 1e9}
            if rf["l2"] is None and k * (4 if storage == "f32" else 2) < 256:
                # rows under 256 B: no L2 ceiling measured for that row size; neither memory level binds
                # (P fits L2 at k = 32 fp16, DRAM carries the triples) -- the A-10 worker clamp does
                # (9.5k ratings in flight x the update's latency)
                row["roofline_bound"] = "latency (A-10 worker clamp; no L2 ceiling measured for %d-B rows)" % (
                    k * (4 if storage == "f32" else 2))
            out[f"C5:k{k}/{storage}"] = row
    out["C5:note"] = "k sweep on the Netflix shape (configs[4]); k = 128 is the headline / hogwild/f32 lines"
    return out


def c3_leg(mf, stream, local, storage, epochs=5):
    return shape_leg(mf, stream, local, storage, "C3",
                     (("hogwild", "hogwild", {}), ("wavefront_cta", "wavefront", {"wave_cta": 1}),
                      ("wavefront_warp", "wavefront", {})), epochs)


def run_partitioned(a, cfg, rank, world, local):
    """N > 1: the partitioned path with NCCL Q rotation, one process per GPU.

    --scaling weak (default): every rank owns a --config-shaped row segment (C2: 480,190 rows, 99M
    samples), so the global problem is m = 480,190 G rows x n = 17,771 columns with 99M G ratings (a
    Hugewiki-like aspect ratio) and per-GPU work is fixed as G grows.  --scaling strong: --config itself
    is split (C4, the Hugewiki shape, at 2/4/8 GPUs).  Each rank generates only its own shard of one
    global planted model (datagen.make_segment)."""
    import torch
    import torch.distributed as dist
    from paper_1610_05838_b200 import mf

    # Test hooks (tests/test_gpu_bench_multirank.py): several ranks on ONE GPU with libmf's NCCL calls
    # served by tests/fake_nccl (LD_PRELOAD) and torch.distributed's own plumbing on gloo.
    backend = os.environ.get("MF_BENCH_DIST_BACKEND", "nccl")
    local = int(os.environ.get("MF_BENCH_DEVICE", local))
    torch.cuda.set_device(local)
    if world == 1:  # --partitioned on one GPU: a 1-rank NCCL job exercising the multi-GPU code path
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend)
    red_dev = "cuda" if backend == "nccl" else "cpu"  # device of the timing reductions
    stream = torch.cuda.current_stream()
    G = world
    m_glob = partition_shape(cfg, G, a.scaling)[0]
    (u, v, r), (tu, tv, tr) = shard(cfg, G, rank, a.scaling)
    N_loc = len(u)
    variant = a.variant if a.variant >= 0 else 0

    def make_ctx():
        # a fresh NCCL unique id per communicator (an id bootstraps exactly one ncclCommInitRank)
        uid = [mf.mf_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        g = mf.MF(m_glob, cfg.n, cfg.k, cfg.alpha, cfg.lam, cfg.seed_init, storage=a.storage, beta=cfg.beta,
                  seed_shuffle=cfg.seed_shuffle, device=local, stream=stream.cuda_stream, variant=variant,
                  workers=a.workers)
        mf.mf_attach_nccl(g.h, uid[0], rank, G)
        return g

    g = make_ctx()
    du, dv, dr = (torch.from_numpy(x).cuda() for x in (u, v, r))
    dtu, dtv, dtr = (torch.from_numpy(x).cuda() for x in (tu, tv, tr))
    g.load(du, dv, dr)
    # the library keeps its own copy; at the Hugewiki shape on few GPUs the staging tensors would otherwise
    # hold 12 B/sample of HBM through the partition layout's sort (R + layout + sort keys + P)
    del du, dv, dr
    torch.cuda.empty_cache()

    def step():
        st = g.epoch("partitioned")
        return st, g.rmse(dtu, dtv, dtr)

    for _ in range(a.warmup):
        step()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    kern, launches = [], 0
    dist.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        e0.record(stream)
        for _ in range(a.steps):
            st, rm = step()
            kern.append(st.kernel_seconds)
            launches += st.launches + 3
        e1.record(stream)
        torch.cuda.synchronize()
    dist.barrier()
    ms = torch.tensor([e0.elapsed_time(e1) / a.steps], device=red_dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms)
    n_tot = torch.tensor([float(N_loc)], device=red_dev)
    dist.all_reduce(n_tot)
    n_tot = float(n_tot)
    value = n_tot / (ms * 1e-3)
    k_s = statistics.mean(kern)
    t_full = load_traffic(a.storage, cfg.name, "hogwild")
    traffic_loc = t_full * N_loc / cfg.n_train if t_full and a.scaling == "strong" else None
    g.close()

    hu, hv, hr = (torch.from_numpy(x).pin_memory() for x in (u, v, r))
    htu, htv, htr = (torch.from_numpy(x).pin_memory() for x in (tu, tv, tr))
    ge = make_ctx()

    def e2e_step():
        ge.load(hu, hv, hr)
        ge.epoch("partitioned")
        return ge.rmse(htu, htv, htr)

    e2e_step()
    dist.barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(a.e2e_steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = torch.tensor([e0.elapsed_time(e1) / a.e2e_steps], device=red_dev)
    dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    ge.close()
    if rank == 0:
        out = {
            "metric": "sgd_updates_per_sec", "value": value, "unit": "updates/s", "n_gpus": G, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": a.scaling,
            "vs_baseline": None, "dtype": "f32", "storage": a.storage, "data": "synthetic",
            "config": workload_config(cfg, G, a.storage, "partitioned", a.scaling),
            "arm": {"workers_per_partition": st.workers, "q_segment_cols": cfg.n // G,
                    "in_flight_per_q_column": st.workers / max(1, cfg.n // G),
                    "note": "accuracy falls with in-flight ratings per Q-segment column (DESIGN.md 5.5)"},
            "test_rmse": rm,
            "roofline": dict(roofline(cfg, a.storage, N_loc, k_s, traffic_loc, "hogwild"),
                             kernel="k_hogwild (rank 0, all launches of the epoch)",
                             traffic_basis="ncu DRAM bytes of the one-GPU batch-Hogwild! launch on this config, "
                                           "scaled to the rank's share of the ratings" if traffic_loc else None),
            "cpu_baseline": None,
            "e2e": {"value": n_tot / (float(e2e_ms) * 1e-3), "unit": "updates/s",
                    "h2d_bytes_per_step": 12 * N_loc * G + 12 * len(tu) * G, "d2h_bytes_per_step": 8 * G,
                    "ms_per_step": float(e2e_ms)},
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
