"""Drives every kernel of libozgpu.so once at small shapes, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool memcheck python tools/sanitize_all.py

Covers: both slicing paths (two-kernel and one-launch queue) and the generic
slicers (int64 / nearest mode), the CTA-pair GEMM with bins, lockstep and the
split-k tail, the B-multicast and plain 1-CTA GEMMs, the fused and folded
epilogues, both exact combines and the sequential combine, the host pipeline,
the kappa scan, the FP64 |A||B| kernel, the integer_gemm tensor and exact
paths, and the pair-planes / int8-slicer debug hooks.  Prints one line per
case; exits non-zero on any library error.  (Development tool; the parity
of these paths is asserted by tests/, not here.)
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2506_11277_b200 as oz  # noqa: E402

CASES = [
    ("default (CTA pair 256x512, bins, lockstep, split-k tail, TMA-stored planes)", {}),
    ("CTA pair 256x256", {"OZGPU_PAIR_N": "256", "OZGPU_BINS": "1"}),
    ("plain plane stores", {"OZGPU_TMA_STORE": "0"}),
    ("4-CTA clusters, B multicast", {"OZGPU_QUAD": "1", "OZGPU_BINS": "1"}),
    ("no lockstep", {"OZGPU_SYNC": "0", "OZGPU_BINS": "1"}),
    ("1-CTA B multicast", {"OZGPU_CTA_PAIR": "0"}),
    ("1-CTA plain", {"OZGPU_CTA_PAIR": "0", "OZGPU_MC": "0", "OZGPU_BINS": "1"}),
    ("fused epilogue", {"OZGPU_EPILOGUE": "fused", "OZGPU_CTA_PAIR": "0"}),
    ("folded combine", {"OZGPU_EPILOGUE": "final", "OZGPU_CTA_PAIR": "0"}),
    ("horner combine", {"OZGPU_COMBINE": "horner"}),
    ("queue slicer", {"OZGPU_SLICE_QUEUE": "1", "OZGPU_SLICE_PANEL_MB": "1"}),
    ("row-blocked planes", {"OZGPU_PLANE_BUDGET_GB": "0.001"}),
]


def main():
    rng = np.random.default_rng(1)
    cfg = oz.MmaConfig.int8_int32()
    m, k, n = 1040, 384, 1100
    a = -0.5 + rng.random((m, k))
    b = (-0.5 + rng.random((k, n))) * np.exp2(rng.integers(-20, 20, size=(k, n)))
    base = None
    for name, env in CASES:
        saved = {key: os.environ.get(key) for key in env}
        os.environ.update(env)
        for sa, sb in [(4, 4), (13, 12), (16, 17)]:
            c = oz.multiply(a, b, cfg, oz.make_plan(cfg, k, sa, sb)).c
            if (sa, sb) == (13, 12):
                if base is None:
                    base = c
                assert np.array_equal(c.view(np.uint64), base.view(np.uint64)), name
        for key, v in saved.items():
            if v is None:
                os.environ.pop(key, None)
            else:
                os.environ[key] = v
        print("ok", name, flush=True)
    for strategy in (0, 1):
        oz.multiply(a[:64], b[:, :70], cfg,
                    oz.make_plan(cfg, k, 5, 6, strategy=oz.Accumulation(strategy)))
    print("ok sequential strategies", flush=True)
    oz.multiply(a[:40], b[:, :50], cfg, oz.make_plan(cfg, k, 5, 5, mode=oz.SliceMode.NEAREST))
    oz.multiply_axpby(1.5, a[:64], b[:, :64], -0.5, a[:64, :64], cfg, oz.make_plan(cfg, k, 6, 6))
    print("ok nearest mode, axpby", flush=True)
    oz.split_rows(a[:33], 7, 5)
    oz.split_cols(b[:, :33], 7, 5, oz.SliceMode.NEAREST)
    oz.split_i8(a, 7, 12, oz.BlockOrientation.ROWS)
    oz.split_i8(b, 7, 12, oz.BlockOrientation.COLUMNS)
    oz.pair_planes(a, b, cfg, oz.make_plan(cfg, k, 13, 12), (0, 16, 0, 16))
    print("ok split hooks, pair planes", flush=True)
    x = rng.integers(-128, 128, size=(300, 256))
    y = rng.integers(-128, 128, size=(256, 200))
    oz.integer_gemm(x, y, cfg)
    try:  # the exact CUDA-core path with the per-MAC overflow check
        oz.integer_gemm(x[:4, :64] // 16 + 120, y[:64, :5] // 16 + 120, oz.MmaConfig(7, 19))
    except oz.MmaOverflowError:
        pass
    print("ok integer_gemm", flush=True)
    oz.scaling_profile(a, b)
    oz.error_bound(a[:64, :96], b[:96, :48], oz.make_plan(cfg, 96, 4, 4))
    print("ok kappa scan, |A||B|", flush=True)
    # the host pipeline (>= 2048 rows, >= 64 MiB)
    big_a = -0.5 + rng.random((2304, 1536))
    big_b = -0.5 + rng.random((1536, 2048))
    oz.multiply(big_a, big_b, cfg, oz.make_plan(cfg, 1536, 6, 6))
    print("ok host pipeline", flush=True)
    # validation tools: exact_gemm (error-free slices + full schedule), metrics
    ex = oz.exact_gemm(a[:96], b[:, :80])
    oz.max_elementwise_error(ex, ex)
    oz.normwise_gemm_error(ex, ex, a[:96], b[:, :80], np.zeros_like(ex), 1.0, 0.0)
    oz.min_exact_slices(a[:50], 7, oz.BlockOrientation.ROWS)
    print("ok exact_gemm, metrics", flush=True)
    # device-resident sharding with the peer-copy path (two contexts on one GPU)
    import torch
    os.environ["OZGPU_MULTI_PEER"] = "1"
    dev = torch.device("cuda:0")
    da, db = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
    dc = torch.empty(m, n, dtype=torch.float64, device=dev)
    st = torch.zeros(2, dtype=torch.int32, device=dev)
    oz.multiply_device_multi(m, n, k, da.data_ptr(), k, db.data_ptr(), n, dc.data_ptr(), n, cfg,
                             oz.make_plan(cfg, k, 6, 6), [0, 0], status_ptr=st.data_ptr())
    torch.cuda.synchronize()
    os.environ.pop("OZGPU_MULTI_PEER")
    print("ok device multi (peer copies)", flush=True)


if __name__ == "__main__":
    main()
