"""Development probe: the end-to-end streamed epoch (mf_epoch_host from pinned host memory) against the raw
host-to-device copy rate, per chunk size (MF_OPT_STREAM_CHUNK)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import datagen  # noqa: E402
from paper_1610_05838_b200 import mf  # noqa: E402


def main():
    cfg = datagen.CONFIGS["C2"]
    (u, v, r), _ = datagen.make(cfg)
    hu, hv, hr = (torch.from_numpy(x).pin_memory() for x in (u, v, r))
    du, dv, dr = (torch.empty_like(x, device="cuda") for x in (hu, hv, hr))
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(2):
        e0.record(s)
        for a, b in ((du, hu), (dv, hv), (dr, hr)):
            a.copy_(b, non_blocking=True)
        e1.record(s)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    nbytes = 12 * len(u)
    print(f"raw H2D {nbytes / 1e9:.2f} GB: {ms:.2f} ms = {nbytes / ms / 1e6:.1f} GB/s", flush=True)
    for chunk in (1 << 21, 1 << 22, 1 << 23, 1 << 24, 1 << 25):
        g = mf.MF(cfg.m, cfg.n, cfg.k, cfg.alpha, cfg.lam, cfg.seed_init, storage="f16", beta=cfg.beta,
                  stream_chunk=chunk, stream=s.cuda_stream)
        g.epoch_host(hu, hv, hr)
        torch.cuda.synchronize()
        e0.record(s)
        for _ in range(3):
            g.epoch_host(hu, hv, hr)
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(f"chunk 2^{chunk.bit_length() - 1}: {ms:.2f} ms per epoch = {len(u) / ms / 1e6:.2f} G updates/s, "
              f"{nbytes / ms / 1e6:.1f} GB/s", flush=True)
        g.close()


if __name__ == "__main__":
    main()
