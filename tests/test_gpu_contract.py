"""C-ABI contract on the GPU: the workspace ordering across streams (the
reference's multiply is called from host thread pools, main.cpp:422,486,557,
and must stay deterministic), operand validation, and
C left untouched when the inputs are rejected (scheme.cpp:223-225)."""
import ctypes

import numpy as np
import pytest

from helpers import bits_equal, mismatch_report, random_matrix, uniform

pytestmark = pytest.mark.gpu


def test_device_calls_on_two_streams_and_host_call_are_ordered(oz, ref):
    """ozgpu_dgemm_device returns without synchronising; two calls on
    different streams with different inputs and plans, followed at once by a
    host-pointer multiply, all share the context's workspace.  Each result must
    equal its own serial result bitwise (eager, graph capture and replays)."""
    import torch
    rng = np.random.default_rng(123)
    cfg = oz.MmaConfig.int8_int32()
    dev = torch.device("cuda:0")
    m, k, n = 1536, 2048, 1280
    a1, b1 = uniform(m, k, rng), uniform(k, n, rng)
    a2, b2 = random_matrix(m, k, rng, -9, 9, 0.01), random_matrix(k, n, rng, -9, 9, 0.01)
    a3, b3 = uniform(700, 900, rng), uniform(900, 650, rng)
    p1, p2, p3 = oz.make_plan(cfg, k, 12, 11), oz.make_plan(cfg, k, 9, 9), oz.make_plan(cfg, 900, 7, 6)
    want1 = oz.multiply(a1, b1, cfg, p1).c
    want2 = oz.multiply(a2, b2, cfg, p2).c
    want3 = oz.multiply(a3, b3, cfg, p3).c
    # anchor the serial results on the reference (corner blocks)
    blocks = [(0, 16, 0, 16), (m - 16, m, n - 16, n)]
    r1, _ = ref.ref_multiply_blocks(a1, b1, 12, 11, blocks, 2)
    for r0, r1_, c0, c1 in blocks:
        assert bits_equal(want1[r0:r1_, c0:c1], r1[r0:r1_, c0:c1])
    s1, s2 = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    A1, B1 = torch.from_numpy(a1).to(dev), torch.from_numpy(b1).to(dev)
    A2, B2 = torch.from_numpy(a2).to(dev), torch.from_numpy(b2).to(dev)
    C1 = torch.empty(m, n, dtype=torch.float64, device=dev)
    C2 = torch.empty(m, n, dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    for it in range(4):  # eager, capture, replay, replay on each stream
        C1.fill_(0.0)
        C2.fill_(0.0)
        torch.cuda.synchronize()
        oz.multiply_device(m, n, k, A1.data_ptr(), k, B1.data_ptr(), n, C1.data_ptr(), n, cfg, p1,
                           stream=s1.cuda_stream)
        oz.multiply_device(m, n, k, A2.data_ptr(), k, B2.data_ptr(), n, C2.data_ptr(), n, cfg, p2,
                           stream=s2.cuda_stream)
        got3 = oz.multiply(a3, b3, cfg, p3).c  # host path on the context's own stream
        torch.cuda.synchronize()
        got1, got2 = C1.cpu().numpy(), C2.cpu().numpy()
        assert bits_equal(got1, want1), (it, mismatch_report(got1, want1))
        assert bits_equal(got2, want2), (it, mismatch_report(got2, want2))
        assert bits_equal(got3, want3), (it, mismatch_report(got3, want3))


def test_operand_validation(oz):
    """lda < k, ldb < n, ldc < n and null pointers are rejected before any
    copy or launch (C-ABI contract; the reference's Matrix carries its shape)."""
    lib = oz._lib
    cfg = oz.MmaConfig.int8_int32()
    plan = oz.make_plan(cfg, 8, 2, 2)._c()
    a = np.ones((4, 8))
    b = np.ones((8, 6))
    c = np.zeros((4, 6))
    ctx = oz._ctx()
    dp = oz._dp
    cases = [(8, 6, 6, "", "ok"), (7, 6, 6, "leading dimension of A", "lda"),
             (8, 5, 6, "leading dimension of B", "ldb"), (8, 6, 5, "leading dimension of C", "ldc")]
    for lda, ldb, ldc, msg, tag in cases:
        rc = lib.ozgpu_dgemm(ctx, 4, 6, 8, dp(a), lda, dp(b), ldb, dp(c), ldc, cfg._c(),
                             ctypes.byref(plan), None)
        if tag == "ok":
            assert rc == 0
        else:
            assert rc == 1 and msg in lib.ozgpu_last_error().decode(), tag
    rc = lib.ozgpu_dgemm(ctx, 4, 6, 8, None, 8, dp(b), 6, dp(c), 6, cfg._c(), ctypes.byref(plan),
                         None)
    assert rc == 1 and "null" in lib.ozgpu_last_error().decode()
    rc = lib.ozgpu_dgemm_device(ctx, 4, 6, 8, None, 8, None, 6, None, 6, cfg._c(),
                                ctypes.byref(plan), None, None, None)
    assert rc == 1 and "null" in lib.ozgpu_last_error().decode()
    # the next valid call is not poisoned by the rejected ones
    assert lib.ozgpu_dgemm(ctx, 4, 6, 8, dp(a), 8, dp(b), 6, dp(c), 6, cfg._c(),
                           ctypes.byref(plan), None) == 0
    assert (c == 8.0).all()


@pytest.mark.parametrize("shape", [(40, 30, 20), (600, 500, 400), (2304, 1536, 2048)])
def test_rejected_inputs_leave_c_untouched(oz, shape):
    """Inf / NaN / -0 inputs raise invalid_argument (scheme.cpp:223-225) and
    the caller's (pageable) C keeps its contents: the unstaged path, and the
    staged pipeline, which unstages C blocks only once the status is read."""
    m, k, n = shape
    cfg = oz.MmaConfig.int8_int32()
    plan = oz.make_plan(cfg, k, 4, 4)
    rng = np.random.default_rng(2)
    a, b = uniform(m, k, rng), uniform(k, n, rng)
    a[m // 2, k // 3] = np.nan
    out = np.full((m, n), 7.25)
    with pytest.raises(oz.InvalidArgument):
        oz.multiply(a, b, cfg, plan, out=out)
    assert (out == 7.25).all()


@pytest.mark.parametrize("slots", [[0, 0], [0, 0, 0], [0, 0, 0, 0]])
def test_sharded_multiply_is_bitwise_identical(oz, ref, slots):
    """ozgpu_dgemm_multi (2-D C tiles over several contexts -- here extra
    contexts on the one GPU this run has, so the tiling, the per-slot
    pipelines and the concurrency are exercised): bitwise the single-context
    result and Diagnostics, incl. a pipelined size, the sequential strategy's
    realized psi, and the input error."""
    rng = np.random.default_rng(len(slots))
    cfg = oz.MmaConfig.int8_int32()
    for (m, k, n), strategy in [((4200, 700, 2600), 2), ((300, 257, 190), 1), ((5, 9, 3), 2)]:
        a = uniform(m, k, rng)
        b = random_matrix(k, n, rng, -12, 12, 0.02)
        plan = oz.make_plan(cfg, k, 9, 8, strategy=oz.Accumulation(strategy))
        want = oz.multiply(a, b, cfg, plan)
        got = oz.multiply(a, b, cfg, plan, devices=slots)
        assert bits_equal(got.c, want.c), (m, k, n, mismatch_report(got.c, want.c))
        assert got.diagnostics == want.diagnostics
    a[2, 2] = np.inf
    with pytest.raises(oz.InvalidArgument, match="finite"):
        oz.multiply(a, b, cfg, plan, devices=slots)


def test_cpp_api_shards_over_ozgpu_devices(oz, ref):
    """The reference's own scheme_test suite, compiled against this library's
    drop-in headers, passes with ozmul::multiply sharding C over two device
    slots (OZGPU_DEVICES=0,0 -> ozgpu_dgemm_multi)."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(ref.REF_PATH), "conf_scheme_test")
    if not os.path.exists(exe):
        pytest.skip("conformance binaries not built")
    env = dict(os.environ, OZGPU_DEVICES="0,0")
    r = subprocess.run([exe], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-2000:])


@pytest.mark.parametrize("peer", [0, 1])
@pytest.mark.parametrize("slots", [[0, 0], [0, 0, 0, 0]])
def test_device_sharded_multiply(oz, slots, peer, monkeypatch):
    """ozgpu_dgemm_device_multi: device-resident A / B / C (strided, lda > k,
    ldb > n, ldc > n) split in 2-D C tiles over extra contexts on the one
    GPU.  peer=1 (OZGPU_MULTI_PEER) treats them as remote, so the panel pulls
    and C-block pushes of the NVLink path run as device-to-device copies.
    Bitwise the single-context result over eager / capture / replay calls,
    ordered on the caller's stream without a host sync, the padding of C
    untouched, and per-block input status."""
    import torch
    monkeypatch.setenv("OZGPU_MULTI_PEER", str(peer))
    rng = np.random.default_rng(7 + len(slots))
    cfg = oz.MmaConfig.int8_int32()
    dev = torch.device("cuda:0")
    m, k, n = 2100, 1100, 1700
    a = uniform(m, k, rng)
    b = random_matrix(k, n, rng, -10, 10, 0.02)
    plan = oz.make_plan(cfg, k, 8, 8)
    want = oz.multiply(a, b, cfg, plan)
    A = torch.zeros(m, k + 40, dtype=torch.float64, device=dev)
    B = torch.zeros(k, n + 24, dtype=torch.float64, device=dev)
    A[:, :k] = torch.from_numpy(a)
    B[:, :n] = torch.from_numpy(b)
    C = torch.full((m, n + 8), 3.5, dtype=torch.float64, device=dev)
    status = torch.full((len(slots),), -1, dtype=torch.int32, device=dev)
    s = torch.cuda.Stream(device=dev)
    torch.cuda.synchronize()
    for it in range(3):
        with torch.cuda.stream(s):
            C[:, :n].fill_(0.0)
        d = oz.multiply_device_multi(m, n, k, A.data_ptr(), k + 40, B.data_ptr(), n + 24,
                                     C.data_ptr(), n + 8, cfg, plan, slots, src_device=0,
                                     stream=s.cuda_stream, status_ptr=status.data_ptr())
        with torch.cuda.stream(s):  # ordered after every block without a host sync
            got = C.clone()
            st = status.clone()
        s.synchronize()
        g = got.cpu().numpy()
        assert bits_equal(np.ascontiguousarray(g[:, :n]), want.c), (it, mismatch_report(g[:, :n], want.c))
        assert (g[:, n:] == 3.5).all()
        assert st.cpu().tolist() == [0] * len(slots)
        assert d == want.diagnostics
    # a NaN in the last row of A dirties only the blocks of the last block row
    A[m - 1, 5] = float("nan")
    oz.multiply_device_multi(m, n, k, A.data_ptr(), k + 40, B.data_ptr(), n + 24, C.data_ptr(),
                             n + 8, cfg, plan, slots, stream=s.cuda_stream,
                             status_ptr=status.data_ptr())
    s.synchronize()
    flags = [v != 0 for v in status.cpu().tolist()]
    assert flags == ([False, True] if len(slots) == 2 else [False, False, True, True])
    # too small to split (m < p_r): one block, every slot written
    status.fill_(-1)
    tiny = torch.from_numpy(uniform(1, k, rng)).to(dev)
    ct = torch.empty(1, n, dtype=torch.float64, device=dev)
    oz.multiply_device_multi(1, n, k, tiny.data_ptr(), k, B.data_ptr(), n + 24, ct.data_ptr(), n,
                             cfg, plan, slots, stream=s.cuda_stream, status_ptr=status.data_ptr())
    s.synchronize()
    assert status.cpu().tolist() == [0] * len(slots)
    want_t = oz.multiply(tiny.cpu().numpy(), b, cfg, plan).c
    assert bits_equal(ct.cpu().numpy(), want_t)


def test_cpp_gemm_fn_hook(tmp_path):
    """ozmul::make_gemm_fn, the GemmFn operator hook (oracle.hpp:117) of the
    C++ drop-in: bitwise the reference callers' hand-built lambda
    (main.cpp:578-582), and a block LU whose Schur updates go through it
    solves its system (tests/native/gemm_fn_test.cpp)."""
    import os
    import subprocess
    from conftest import ROOT
    lib = os.path.join(ROOT, "paper_2506_11277_b200", "lib")
    exe = str(tmp_path / "gemm_fn_test")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "native", "gemm_fn_test.cpp"),
                    os.path.join(lib, "libozgpu.so"), "-Wl,-rpath," + lib, "-o", exe], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.startswith("ok"), r.stdout


def test_python_gemm_fn_hook(oz):
    """The Python mirror of the hook: gemm_fn(cfg, sa, sb) makes its plan per
    call from the operands' inner dimension, bitwise multiply() with that plan."""
    rng = np.random.default_rng(17)
    cfg = oz.MmaConfig.int8_int32()
    fn = oz.gemm_fn(cfg, 9, 8)
    for m, k, n in [(300, 16, 290), (129, 700, 65), (1, 1, 1)]:
        x, y = uniform(m, k, rng), uniform(k, n, rng)
        want = oz.multiply(x, y, cfg, oz.make_plan(cfg, k, 9, 8)).c
        assert bits_equal(fn(x, y), want), (m, k, n)
