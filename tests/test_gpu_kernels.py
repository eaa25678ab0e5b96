"""Kernel-level numerics on the B200, each kernel called through the C ABI and
compared with a plain PyTorch fp32 restatement of the same op (or, for the
integer kernels, bit-exactly with the oracle)."""

import ctypes as C
import math
import random

import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2512_15834_b200.modelcfg import ModelShape  # noqa: E402


@pytest.fixture(scope="module")
def lib():
    from paper_2512_15834_b200.runtime import lib as L

    L.load()
    return L


def P(t):
    return C.c_void_p(0 if t is None else t.data_ptr())


def stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def rel(a, b):
    return float((a.float() - b.float()).norm() / b.float().norm().clamp_min(1e-12))


@pytest.mark.parametrize("M,N,K", [(1, 256, 256), (7, 384, 512), (32, 6144, 4096), (32, 4096, 14336),
                                   (100, 1000, 256), (300, 640, 1024), (2048, 1024, 4096), (17, 128256, 256)])
def test_gemm_bf16(lib, M, N, K):
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N + K)
    a = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    w = (0.05 * torch.randn(N, K, device="cuda", generator=g)).to(torch.bfloat16)
    c = torch.full((M, N), float("nan"), device="cuda")
    lib.call("stb_gemm_bf16", P(a), K, P(w), K, P(c), N, M, N, K, 0, 0, stream())
    ref = a.float() @ w.float().T
    torch.cuda.synchronize()
    assert rel(c, ref) < 2e-5


@pytest.mark.parametrize("M,N,K", [(1, 256, 256), (32, 6144, 4096), (64, 4096, 14336), (300, 640, 1024)])
def test_gemm_c_zeroed(lib, M, N, K):
    """STB_GEMM_C_ZEROED: a stream-K GEMM accumulates into a caller-zeroed C (no memset,
    no grid barrier); tile-mode shapes ignore the flag."""
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    w = (0.05 * torch.randn(N, K, device="cuda")).to(torch.bfloat16)
    c = torch.zeros(M, N, device="cuda")
    for _ in range(3):  # repeated launches stay exact because the caller re-zeroes
        lib.call("stb_gemm_bf16", P(a), K, P(w), K, P(c), N, M, N, K, 0, 1, stream())
        ref = a.float() @ w.float().T
        assert rel(c, ref) < 2e-5
        c.zero_()
    lib.load().stb_gemm_is_stream.restype  # exported
    assert lib.load().stb_gemm_is_stream(32, 6144, 4096) in (0, 1)


@pytest.mark.parametrize("M,F,K", [(300, 1024, 512), (608, 2048, 1024), (2080, 512, 256), (200, 14336, 4096)])
def test_gemm_silu_fused(lib, M, F, K):
    """STB_GEMM_SILU_MUL: tile-schedule epilogue emits bf16 silu(gate)*up from interleaved
    (gate, up) weight rows — bit-identical to the fp32 GEMM followed by stb_silu_mul."""
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    w = (0.05 * torch.randn(2 * F, K, device="cuda")).to(torch.bfloat16)
    act = torch.full((M, F), float("nan"), device="cuda").to(torch.bfloat16)
    lib.call("stb_gemm_bf16", P(a), K, P(w), K, P(act), F, M, 2 * F, K, 1, 2, stream())
    c = torch.zeros(M, 2 * F, device="cuda")
    lib.call("stb_gemm_bf16", P(a), K, P(w), K, P(c), 2 * F, M, 2 * F, K, 1, 0, stream())
    ref = torch.empty(M, F, device="cuda", dtype=torch.bfloat16)
    lib.call("stb_silu_mul", P(c), P(ref), M, F, 0, stream())
    torch.cuda.synchronize()
    assert torch.equal(act, ref)
    full = a.float() @ w.float().T
    assert rel(act, torch.nn.functional.silu(full[:, 0::2]) * full[:, 1::2]) < 1e-2
    if lib.load().stb_gemm_is_stream(32, 2 * F, K):  # fused epilogue refuses the stream-K schedule
        with pytest.raises(Exception):
            lib.call("stb_gemm_bf16", P(a), K, P(w), K, P(act), F, 32, 2 * F, K, 0, 2, stream())


def test_gemm_explicit_split(lib):
    M, N, K = 32, 512, 4096
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    w = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    ref = a.float() @ w.float().T
    for split in (1, 2, 5, 64, 148):
        c = torch.full((M, N), float("nan"), device="cuda")
        lib.call("stb_gemm_bf16", P(a), K, P(w), K, P(c), N, M, N, K, split, 0, stream())
        assert rel(c, ref) < 2e-5, split


def _tiled(lib, w):
    N, K = w.shape
    t = torch.full((lib.load().stb_weight_tiled_elems(N, K),), float("nan"), device="cuda").to(torch.bfloat16)
    lib.call("stb_weight_tile", P(w), w.stride(0), N, K, P(t), stream())
    return t


def test_weight_tile_layout(lib):
    """stb_weight_tile: tile (n, k) contiguous, rows of 64, 16-byte chunk c of row r at c ^ (r & 7),
    zero padding past N and K (restated here in torch)."""
    N, K = 200, 72
    w = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    t = _tiled(lib, w)
    pad = torch.zeros(256, 128, device="cuda", dtype=torch.bfloat16)
    pad[:N, :K] = w
    ref = pad.view(2, 128, 2, 8, 8).permute(0, 2, 1, 3, 4).clone()  # [nt][kt][r][c][e]
    r = torch.arange(128, device="cuda").view(128, 1)
    perm = torch.arange(8, device="cuda").view(1, 8) ^ (r & 7)          # physical chunk -> logical
    ref = torch.gather(ref, 3, perm.view(1, 1, 128, 8, 1).expand(2, 2, 128, 8, 8))
    assert torch.equal(t, ref.reshape(-1))


@pytest.mark.parametrize("M,N,K", [(1, 256, 256), (32, 6144, 4096), (32, 4096, 14336), (17, 130, 200),
                                   (300, 640, 1024), (608, 28672, 4096),
                                   (32, 128256, 4096), (65, 28672, 4096)])  # C2 LM head, verify-step gate-up
def test_gemm_w_tiled(lib, M, N, K):
    """STB_GEMM_W_TILED: the same products from the tiled weight layout (both schedules)."""
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    w = (0.05 * torch.randn(N, K, device="cuda")).to(torch.bfloat16)
    t = _tiled(lib, w)
    ref = a.float() @ w.float().T
    for split in (0, 1, 7):
        c = torch.full((M, N), float("nan"), device="cuda")
        lib.call("stb_gemm_bf16", P(a), K, P(t), 0, P(c), N, M, N, K, split, 4, stream())
        assert rel(c, ref) < 2e-5, split
    if N % 2 == 0:  # fused SiLU epilogue from tiled weights
        act = torch.empty(M, N // 2, device="cuda", dtype=torch.bfloat16)
        lib.call("stb_gemm_bf16", P(a), K, P(t), 0, P(act), N // 2, M, N, K, 1, 2 | 4, stream())
        want = torch.nn.functional.silu(ref[:, 0::2]) * ref[:, 1::2]
        assert rel(act, want) < 1e-2


@pytest.mark.parametrize("M,N,K,tiled", [(608, 4096, 14336, True), (608, 4096, 14336, False), (608, 28672, 4096, True),
                                         (2080, 9216, 4096, False), (700, 10240, 2048, True)])
def test_gemm_pair_cta_group2(lib, M, N, K, tiled):
    """K5 pair kernel (CTA pairs, tcgen05.mma.cta_group::2): prefill-shaped products with
    N > 8192 or K >= 8192 take it; plain stores and the SiLU-gate epilogue, ragged M."""
    from paper_2512_15834_b200.runtime.decoder import TiledWeight

    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    a = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    w = (0.05 * torch.randn(N, K, device="cuda", generator=g)).to(torch.bfloat16)
    wt, ldw, fl = (TiledWeight(w), 0, 4) if tiled else (w, K, 0)
    assert not lib.load().stb_gemm_is_stream(M, N, K)  # whole tiles: pair-eligible shapes
    ref = a.float() @ w.float().T
    c = torch.full((M, N), float("nan"), device="cuda")
    lib.call("stb_gemm_bf16", P(a), K, P(wt), ldw, P(c), N, M, N, K, 0, fl, stream())
    torch.cuda.synchronize()
    assert rel(c, ref) < 2e-5
    act = torch.full((M, N // 2), float("nan"), device="cuda").to(torch.bfloat16)
    lib.call("stb_gemm_bf16", P(a), K, P(wt), ldw, P(act), N // 2, M, N, K, 0, fl | 2, stream())
    want = torch.nn.functional.silu(ref[:, 0::2]) * ref[:, 1::2]
    assert rel(act, want) < 1e-2


def _epi(**kw):
    from paper_2512_15834_b200.runtime.decoder import GemmEpi

    return GemmEpi(**kw)


@pytest.mark.parametrize("M", [1, 32, 100, 300])
def test_gemm_fused_silu_resid(lib, M):
    """STB_EPI_SILU with the input-row RMSNorm scale, and STB_EPI_RESID, vs torch fp32; the
    workspace is left zeroed (stream-K fixups clear what they reduce)."""
    from paper_2512_15834_b200.runtime.decoder import TiledWeight

    K, F, D = 1024, 640, 512
    g = torch.Generator(device="cuda").manual_seed(M)
    a = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    ss = (a.float() ** 2).sum(1) * torch.rand(M, device="cuda", generator=g) * 2
    wgu = TiledWeight((0.05 * torch.randn(2 * F, K, device="cuda", generator=g)).to(torch.bfloat16))
    work = torch.zeros(M, 2 * F, device="cuda")
    act = torch.full((M, F), float("nan"), device="cuda").to(torch.bfloat16)
    ss4 = torch.zeros(M, 4, device="cuda")  # partial sums of squares: the total in slot 0
    ss4[:, 0] = ss
    e = _epi(kind=1, ss_in=ss4.data_ptr(), ss_parts=4, inv_dim=1.0 / K, eps=1e-5, out=act.data_ptr(), ldo=F)
    fn = lib.load().stb_gemm_bf16_fused
    # M <= 128: stream-K (every tile split over ~16 CTAs: the ticket fixup); M = 300: whole tiles
    rc = fn(P(a), K, P(wgu), 0, P(work), 2 * F, M, 2 * F, K, 4, C.byref(e), stream())
    assert rc == 0, lib.load().stb_last_error()
    full = a.float() @ TiledWeight_ref(wgu).T
    full = full * torch.rsqrt(ss / K + 1e-5)[:, None]
    want = torch.nn.functional.silu(full[:, 0::2]) * full[:, 1::2]
    torch.cuda.synchronize()
    assert rel(act, want) < 1e-2
    assert not work.any()
    # RESID
    wo = (0.05 * torch.randn(D, K, device="cuda", generator=g)).to(torch.bfloat16)
    two = TiledWeight(wo)
    x = torch.randn(M, D, device="cuda", generator=g)
    x0 = x.clone()
    xb = torch.empty(M, D, device="cuda", dtype=torch.bfloat16)
    sso = torch.full((M, D // 128), float("nan"), device="cuda")
    workd = torch.zeros(M, D, device="cuda")
    e = _epi(kind=3, out=xb.data_ptr(), ldo=D, x=x.data_ptr(), ldx=D, ss_out=sso.data_ptr(), ss_parts=D // 128)
    rc = fn(P(a), K, P(two), 0, P(workd), D, M, D, K, 4, C.byref(e), stream())
    assert rc == 0, lib.load().stb_last_error()
    xr = x0 + a.float() @ wo.float().T
    torch.cuda.synchronize()
    assert rel(x, xr) < 1e-5
    assert torch.equal(xb, x.to(torch.bfloat16))
    assert torch.allclose(sso, (xr ** 2).view(M, D // 128, 128).sum(2), rtol=1e-4)  # per 128-feature tile
    assert not workd.any()


def TiledWeight_ref(tw):
    """fp32 [N][K] from a TiledWeight (inverse of stb_weight_tile)."""
    N, K = tw.N, tw.K
    nt, kt = -(-N // 128), -(-K // 64)
    t = tw.t.view(nt, kt, 128, 8, 8)
    r = torch.arange(128, device="cuda").view(128, 1)
    inv = torch.arange(8, device="cuda").view(1, 8) ^ (r & 7)   # logical chunk -> physical (an involution)
    t = torch.gather(t, 3, inv.view(1, 1, 128, 8, 1).expand(nt, kt, 128, 8, 8))
    return t.permute(0, 2, 1, 3, 4).reshape(nt * 128, kt * 64)[:N, :K].float()


@pytest.mark.parametrize("qk_norm", [False, True])
@pytest.mark.parametrize("d_head,n_q,n_kv", [(128, 8, 2), (64, 4, 2)])
@pytest.mark.parametrize("M", [3, 32, 200])
def test_gemm_fused_qkv(lib, qk_norm, d_head, n_q, n_kv, M):
    """STB_EPI_QKV: input-row RMSNorm scale, (qk-norm,) RoPE, q out and K/V commit into the
    pool — equal to the unfused GEMM + stb_qkv_norm_rope_commit."""
    from paper_2512_15834_b200.runtime.decoder import TiledWeight

    shape = ModelShape("t", 1, 512, n_q, n_kv, d_head, 64, 64, rope_theta=10000.0, rms_eps=1e-6, qk_norm=qk_norm)
    K, N = 512, (n_q + 2 * n_kv) * d_head
    g = torch.Generator(device="cuda").manual_seed(M * 3 + d_head)
    a = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    ss = (a.float() ** 2).sum(1)
    w = (0.05 * torch.randn(N, K, device="cuda", generator=g)).to(torch.bfloat16)
    tw = TiledWeight(w)
    qn = (1.0 + 0.1 * torch.randn(d_head, device="cuda", generator=g)).to(torch.bfloat16)
    kn = (1.0 + 0.1 * torch.randn(d_head, device="cuda", generator=g)).to(torch.bfloat16)
    ctx0 = 40
    pos = torch.arange(ctx0, ctx0 + M, dtype=torch.int32, device="cuda")
    slot_of = torch.zeros(M, dtype=torch.int32, device="cuda")
    pools = []
    for _ in range(2):
        pool = _pool(lib, shape)
        pool.reserve(0, ctx0 + M)
        pool.sync(torch.cuda.current_stream().cuda_stream)
        pools.append(pool)
    # fused
    q1 = torch.zeros(M, n_q * d_head, device="cuda", dtype=torch.bfloat16)
    work = torch.zeros(M, N, device="cuda")
    ss4 = torch.zeros(M, 4, device="cuda")
    ss4[:, 1] = ss
    e = _epi(kind=2, ss_in=ss4.data_ptr(), ss_parts=4, inv_dim=1.0 / K, eps=1e-6, out=q1.data_ptr(), ldo=n_q * d_head,
             pool=pools[0].h.value, layer=0, n_q=n_q, slot_of=slot_of.data_ptr(), pos_of=pos.data_ptr(),
             rope_theta=10000.0, q_norm=qn.data_ptr() if qk_norm else None, k_norm=kn.data_ptr() if qk_norm else None,
             qk_eps=1e-6)
    rc = lib.load().stb_gemm_bf16_fused(P(a), K, P(tw), 0, P(work), N, M, N, K, 4, C.byref(e), stream())
    assert rc == 0, lib.load().stb_last_error()
    # unfused reference: scaled fp32 GEMM -> stb_qkv_norm_rope_commit
    qkv = (a.float() @ w.float().T) * torch.rsqrt(ss / K + 1e-6)[:, None]
    q2 = torch.zeros_like(q1)
    lib.call("stb_qkv_norm_rope_commit", pools[1].h, 0, P(qkv), P(q2), P(slot_of), P(pos), M, n_q, 10000.0,
             P(qn) if qk_norm else None, P(kn) if qk_norm else None, 1e-6, 0, stream())
    torch.cuda.synchronize()
    assert not work.any()
    assert rel(q1, q2) < 1e-2
    k1, v1 = _dense_kv(pools[0], 0, 0, ctx0 + M, shape)
    k2, v2 = _dense_kv(pools[1], 0, 0, ctx0 + M, shape)
    assert rel(k1[ctx0:], k2[ctx0:]) < 1e-2 and rel(v1[ctx0:], v2[ctx0:]) < 1e-2


def test_embed_prep(lib):
    V, d, n, parts = 300, 512, 37, 4
    table = torch.randn(V, d, device="cuda").to(torch.bfloat16)
    ids = torch.randint(0, V, (n,), device="cuda", dtype=torch.int32)
    x = torch.empty(n, d, device="cuda")
    xb = torch.empty(n, d, device="cuda", dtype=torch.bfloat16)
    ss = torch.full((n + 3, parts), 7.0, device="cuda")
    lib.call("stb_embed_prep", P(ids), P(table), P(x), P(xb), P(ss), parts, n, d, stream())
    ref = table[ids.long()].float()
    assert torch.equal(x, ref) and torch.equal(xb, table[ids.long()])
    assert torch.allclose(ss[:n, 0], (ref ** 2).sum(1), rtol=1e-5)
    assert not ss[:n, 1:].any() and (ss[n:] == 7.0).all()


def _pool(lib, shape, nb=256, slots=64, bps=512):
    from paper_2512_15834_b200.runtime.decoder import KVPool

    return KVPool(shape, nb, slots, bps)


def test_allocator_matches_oracle(lib):
    from oracle.kv_alloc import LifoAllocator

    shape = ModelShape("t", 1, 64, 1, 1, 64, 64, 64)
    pool = _pool(lib, shape, nb=200, slots=8, bps=64)
    ref = LifoAllocator(200)
    rng = random.Random(3)
    for _ in range(2000):
        slot = rng.randrange(8)
        op = rng.choice(["res", "res", "trunc", "rel"])
        n = rng.randrange(0, 300)
        if op == "res":
            need = -(-n // 16) - len(ref.blocks(slot))
            if need > len(ref.free):
                continue
            pool.reserve(slot, n)
            ref.reserve(slot, n)
        elif op == "trunc":
            pool.truncate(slot, n)
            ref.truncate(slot, n)
        else:
            pool.release(slot)
            ref.release(slot)
        assert pool.blocks(slot) == ref.blocks(slot)
    assert pool.free_blocks() == len(ref.free)


class _Raw:
    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<u2", "data": (ptr, False), "version": 3}


def _view(ptr, n):
    """Zero-copy bf16 view of n elements of library-owned device memory."""
    return torch.as_tensor(_Raw(ptr, n), device="cuda").view(torch.bfloat16)


def _dense_kv(pool, layer, slot, n, shape):
    """Gather a slot's first n rows from the pool via the block table (torch)."""
    kp, vp = pool.layer_ptrs(layer)
    nb = pool.num_blocks
    per = nb * shape.n_kv * 16 * shape.d_head
    torch.cuda.synchronize()
    kbuf = _view(kp, per)
    vbuf = _view(vp, per)
    # pages are pre-swizzled (csrc/pool.cuh kv_phys_chunk): logical chunk c of row r is
    # stored at chunk (c & ~7) | ((c ^ r) & 7)
    ch = shape.d_head // 8
    perm = torch.tensor([[(c & ~7) | ((c ^ r) & 7) for c in range(ch)] for r in range(16)], device="cuda")
    idx = perm.view(1, 1, 16, ch, 1).expand(nb, shape.n_kv, 16, ch, 8)
    k = kbuf.view(nb, shape.n_kv, 16, ch, 8).gather(3, idx).view(nb, shape.n_kv, 16, shape.d_head)
    v = vbuf.view(nb, shape.n_kv, 16, ch, 8).gather(3, idx).view(nb, shape.n_kv, 16, shape.d_head)
    blocks = torch.tensor(pool.blocks(slot), device="cuda", dtype=torch.long)
    kd = k[blocks].permute(0, 2, 1, 3).reshape(-1, shape.n_kv, shape.d_head)[:n]
    vd = v[blocks].permute(0, 2, 1, 3).reshape(-1, shape.n_kv, shape.d_head)[:n]
    return kd.clone(), vd.clone()


def _fill_pool(lib, pool, shape, ctxs, seed=0):
    """Commit random K/V rows for slots 0..len(ctxs)-1 with stb_kv_commit; returns dense copies."""
    g = torch.Generator(device="cuda").manual_seed(seed)
    dense = []
    for s, n in enumerate(ctxs):
        pool.reserve(s, n)
    pool.sync(torch.cuda.current_stream().cuda_stream)
    for s, n in enumerate(ctxs):
        k = torch.randn(n, shape.kv_dim, device="cuda", generator=g).to(torch.bfloat16)
        v = torch.randn(n, shape.kv_dim, device="cuda", generator=g).to(torch.bfloat16)
        slot_of = torch.full((n,), s, dtype=torch.int32, device="cuda")
        pos = torch.arange(n, dtype=torch.int32, device="cuda")
        for layer in range(shape.layers):
            lib.call("stb_kv_commit", pool.h, layer, P(k), P(v), shape.kv_dim, P(slot_of), P(pos), n, stream())
        dense.append((k.view(n, shape.n_kv, shape.d_head), v.view(n, shape.n_kv, shape.d_head)))
    return dense


def test_kv_commit_roundtrip(lib):
    shape = ModelShape("t", 2, 256, 4, 2, 64, 64, 64)
    pool = _pool(lib, shape)
    dense = _fill_pool(lib, pool, shape, [1, 15, 16, 17, 100])
    for s, (k, v) in enumerate(dense):
        for layer in range(2):
            kd, vd = _dense_kv(pool, layer, s, k.shape[0], shape)
            assert torch.equal(kd, k) and torch.equal(vd, v)


def _ref_attn(q, k, v, qpos, scale):
    # q [n, H, D] fp32, k/v [ctx, G, D]; causal: key j visible iff j <= qpos[i]
    H, G = q.shape[1], k.shape[1]
    kk = k.float().repeat_interleave(H // G, dim=1)
    vv = v.float().repeat_interleave(H // G, dim=1)
    s = torch.einsum("nhd,chd->hnc", q.float(), kk) * scale
    mask = torch.arange(k.shape[0], device=q.device)[None, :] > qpos[:, None]
    s = s.masked_fill(mask[None], float("-inf"))
    return torch.einsum("hnc,chd->nhd", torch.softmax(s, -1), vv)


SHAPES = [ModelShape("llama-ish", 1, 4096, 32, 8, 128, 64, 64), ModelShape("tiny", 1, 256, 4, 2, 64, 64, 64),
          ModelShape("qwen-ish", 1, 5120, 64, 8, 128, 64, 64)]


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: s.name)
@pytest.mark.parametrize("ctxs", [[1], [5, 16, 17, 33], [4096] * 4 + [100, 2500], [700] * 32, [8000], [8000, 2]])
def test_attn_decode(lib, shape, ctxs):
    pool = _pool(lib, shape, nb=sum(-(-c // 16) for c in ctxs) + 8, slots=len(ctxs), bps=512)
    dense = _fill_pool(lib, pool, shape, ctxs, seed=len(ctxs))
    B = len(ctxs)
    q = torch.randn(B, shape.n_q, shape.d_head, device="cuda").to(torch.bfloat16)
    out = torch.empty_like(q)
    slots = torch.arange(B, dtype=torch.int32, device="cuda")
    ctx = torch.tensor(ctxs, dtype=torch.int32, device="cuda")
    ws = torch.zeros(-(-lib.load().stb_attn_decode_workspace(B, shape.n_q, shape.n_kv, shape.d_head) // 4), device="cuda")
    scale = 1 / math.sqrt(shape.d_head)
    lib.call("stb_attn_decode", pool.h, 0, P(q), P(out), P(slots), P(ctx), B, shape.n_q, scale, max(ctxs), P(ws),
             stream())
    for b, (k, v) in enumerate(dense):
        ref = _ref_attn(q[b:b + 1], k, v, torch.tensor([ctxs[b] - 1], device="cuda"), scale)
        assert rel(out[b:b + 1], ref) < 1e-2, b


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: s.name)
@pytest.mark.parametrize("case", [
    ([700] * 3, [(33, 2984)]),                 # C2 verify pass riding with decode rows
    ([5, 16, 17], [(1, 1), (4, 10), (21, 33)]),  # ragged runs, a 1-query run, a run that is its whole context
    ([], [(40, 4096), (33, 100)]),             # runs only (no decode rows)
    ([8000] * 2, [(17, 8017), (2, 20)]),       # long context, split pairs merged by the ticket warp
])
def test_attn_decode_multi_query(lib, shape, case):
    """stb_attn_decode_mq: decode rows (1-query entries) and short runs folded into K3 as multi-query
    entries (16 / group queries per 16-row tile, causal inside the run) vs torch fp32."""
    dec_ctxs, runs = case
    G = shape.n_q // shape.n_kv
    qe = 16 // G
    ctxs = dec_ctxs + [c for _, c in runs]
    pool = _pool(lib, shape, nb=sum(-(-c // 16) for c in ctxs) + 8, slots=len(ctxs), bps=600)
    dense = _fill_pool(lib, pool, shape, ctxs, seed=11)
    B = len(dec_ctxs)
    T = B + sum(n for n, _ in runs)
    q = torch.randn(T, shape.n_q, shape.d_head, device="cuda").to(torch.bfloat16)
    out = torch.full_like(q, float("nan"))
    e_slot, e_ctx, e_row, e_nq = list(range(B)), list(dec_ctxs), list(range(B)), [1] * B
    row = B
    for r, (n, c) in enumerate(runs):
        for j in range(0, n, qe):
            nq = min(qe, n - j)
            e_slot.append(B + r)
            e_ctx.append(c - n + j + nq)
            e_row.append(row + j)
            e_nq.append(nq)
        row += n
    t = lambda a: torch.tensor(a, dtype=torch.int32, device="cuda")  # noqa: E731
    E = len(e_slot)
    ws = torch.zeros(-(-lib.load().stb_attn_decode_workspace(E, shape.n_q, shape.n_kv, shape.d_head) // 4),
                     device="cuda")
    scale = 1 / math.sqrt(shape.d_head)
    meta = [t(a) for a in (e_slot, e_ctx, e_row, e_nq)]  # kept alive until the launches complete
    lib.call("stb_attn_decode_mq", pool.h, 0, P(q), P(out), *[P(a) for a in meta], E, shape.n_q, scale, max(ctxs),
             P(ws), stream())
    for b in range(B):
        k, v = dense[b]
        ref = _ref_attn(q[b:b + 1], k, v, torch.tensor([dec_ctxs[b] - 1], device="cuda"), scale)
        assert rel(out[b:b + 1], ref) < 1e-2, ("decode", b)
    row = B
    for r, (n, c) in enumerate(runs):
        k, v = dense[B + r]
        ref = _ref_attn(q[row:row + n], k, v, torch.arange(c - n, c, device="cuda"), scale)
        assert rel(out[row:row + n], ref) < 1e-2, ("run", r)
        row += n
    assert torch.isfinite(out.float()).all()  # every row written
    # the ticket region is left zeroed (graph-safe): a second launch gives the same result
    out2 = torch.full_like(q, float("nan"))
    lib.call("stb_attn_decode_mq", pool.h, 0, P(q), P(out2), *[P(a) for a in meta], E, shape.n_q, scale, max(ctxs),
             P(ws), stream())
    assert rel(out2, out) < 1e-3


@pytest.mark.parametrize("shape", SHAPES[:2], ids=lambda s: s.name)
@pytest.mark.parametrize("mq", [False, True], ids=["decode", "multi_query"])
@pytest.mark.parametrize("ctxs", [[5, 16, 17, 33], [700] * 32, [4096] * 4 + [100, 2500], [8000, 2]])
def test_attn_decode_planned(lib, shape, mq, ctxs):
    """stb_attn_decode_planned: the partition layer 0 stores (plan_mode 1) and the later layers load
    (plan_mode 2) is the one each launch computes itself (plan_mode 0): bit-identical outputs, for
    several "layers" (fresh q each) of one step, then a step with other contexts re-planned."""
    G = shape.n_q // shape.n_kv
    B = len(ctxs)
    pool = _pool(lib, shape, nb=sum(-(-c // 16) for c in ctxs) * 2 + 8, slots=B, bps=600)
    _fill_pool(lib, pool, shape, ctxs, seed=5)
    t = lambda a: torch.tensor(a, dtype=torch.int32, device="cuda")  # noqa: E731
    ws = torch.zeros(-(-lib.load().stb_attn_decode_workspace(2 * B, shape.n_q, shape.n_kv, shape.d_head) // 4),
                     device="cuda")
    scale = 1 / math.sqrt(shape.d_head)

    def step(cl, layers=3):
        if mq:  # every entry a 1..16/G-query run ending at its context
            nq = [1 + (b % (16 // G)) for b in range(B)]
            rows = [sum(nq[:b]) for b in range(B)]
            meta = [t(list(range(B))), t(cl), t(rows), t(nq)]
            T = sum(nq)
        else:
            meta = [t(list(range(B))), t(cl), None, None]
            T = B
        for layer in range(layers):
            q = torch.randn(T, shape.n_q, shape.d_head, device="cuda").to(torch.bfloat16)
            outs = []
            for mode in (0, 1 if layer == 0 else 2):
                out = torch.full_like(q, float("nan"))
                lib.call("stb_attn_decode_planned", pool.h, 0, P(q), P(out), *[P(a) for a in meta], B, shape.n_q,
                         scale, max(cl), mode, P(ws), stream())
                outs.append(out)
            torch.cuda.synchronize()
            assert torch.isfinite(outs[0].float()).all()
            assert torch.equal(outs[0], outs[1]), layer

    step(ctxs)
    step([max(1, c // 2) for c in ctxs])  # a new step: layer 0 re-plans
    tickets = ws.view(torch.int32)[-(2 * B * shape.n_kv + 64):]
    assert int(tickets.abs().sum()) == 0


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: s.name)
@pytest.mark.parametrize("runs", [[(1, 1)], [(4, 10), (21, 33)], [(300, 300), (33, 1200), (7, 8)],
                                  [(996, 3044), (33, 2174)]])  # C2 trace: ragged ingest + verify
@pytest.mark.parametrize("amp", [1.0, 40.0], ids=["unit", "spiky"])
def test_attn_prefill(lib, shape, runs, amp):
    # amp scales q: "spiky" scores span hundreds of log2 units, exercising the lazy
    # rescale and the clamped FMA-pipe exponentials
    # runs: (n new queries, ctx incl. them)
    ctxs = [c for _, c in runs]
    pool = _pool(lib, shape, nb=sum(-(-c // 16) for c in ctxs) + 8, slots=len(runs), bps=512)
    dense = _fill_pool(lib, pool, shape, ctxs, seed=7)
    T = sum(n for n, _ in runs)
    q = (torch.randn(T, shape.n_q, shape.d_head, device="cuda") * amp).to(torch.bfloat16)
    out = torch.full_like(q, float("nan"))
    qs = [0]
    for n, _ in runs:
        qs.append(qs[-1] + n)
    slots = torch.arange(len(runs), dtype=torch.int32, device="cuda")
    qstart = torch.tensor(qs, dtype=torch.int32, device="cuda")
    ctx = torch.tensor(ctxs, dtype=torch.int32, device="cuda")
    scale = 1 / math.sqrt(shape.d_head)
    lib.call("stb_attn_prefill", pool.h, 0, P(q), P(out), P(slots), P(qstart), P(ctx), len(runs), T, shape.n_q,
             scale, max(n for n, _ in runs), stream())
    for s, ((n, c), (k, v)) in enumerate(zip(runs, dense)):
        qpos = torch.arange(c - n, c, device="cuda")
        ref = _ref_attn(q[qs[s]:qs[s + 1]], k, v, qpos, scale)
        assert rel(out[qs[s]:qs[s + 1]], ref) < 1e-2, s


def _ref_attn_chunked(q, k, v, qpos, scale):
    """_ref_attn one kv head (and its query-head group) at a time: bounds the fp32 score
    tensor at 32k contexts."""
    rep = q.shape[1] // k.shape[1]
    return torch.cat([_ref_attn(q[:, g * rep:(g + 1) * rep], k[:, g:g + 1], v[:, g:g + 1], qpos, scale)
                      for g in range(k.shape[1])], dim=1)


@pytest.mark.parametrize("shape", [SHAPES[0], SHAPES[2]], ids=lambda s: s.name)
def test_attn_long_context_c5(lib, shape):
    """Config C5 (KV pressure): a 2048-token tool output appended in place after a 32,768-token
    resident context (K2), then decode over 32k+ contexts of several sequences (K3)."""
    ctxs = [32768 + 2048, 32768 + 7, 33000]
    pool = _pool(lib, shape, nb=sum(-(-c // 16) for c in ctxs) + 8, slots=len(ctxs), bps=2304)
    dense = _fill_pool(lib, pool, shape, ctxs, seed=5)
    scale = 1 / math.sqrt(shape.d_head)
    # K2: the ingest run of sequence 0
    n = 2048
    q = torch.randn(n, shape.n_q, shape.d_head, device="cuda").to(torch.bfloat16)
    out = torch.full_like(q, float("nan"))
    slot0 = torch.zeros(1, dtype=torch.int32, device="cuda")  # kept alive: the launch reads them
    qstart = torch.tensor([0, n], dtype=torch.int32, device="cuda")
    ctx0 = torch.tensor([ctxs[0]], dtype=torch.int32, device="cuda")
    lib.call("stb_attn_prefill", pool.h, 0, P(q), P(out), P(slot0), P(qstart), P(ctx0), 1, n, shape.n_q, scale, n,
             stream())
    k0, v0 = dense[0]
    ref = _ref_attn_chunked(q, k0, v0, torch.arange(ctxs[0] - n, ctxs[0], device="cuda"), scale)
    assert rel(out, ref) < 1e-2
    # K3: one decode query per sequence at its full context
    B = len(ctxs)
    qd = torch.randn(B, shape.n_q, shape.d_head, device="cuda").to(torch.bfloat16)
    od = torch.empty_like(qd)
    ws = torch.zeros(-(-lib.load().stb_attn_decode_workspace(B, shape.n_q, shape.n_kv, shape.d_head) // 4), device="cuda")
    slots = torch.arange(B, dtype=torch.int32, device="cuda")
    ctx = torch.tensor(ctxs, dtype=torch.int32, device="cuda")
    lib.call("stb_attn_decode", pool.h, 0, P(qd), P(od), P(slots), P(ctx), B, shape.n_q, scale, 0, P(ws), stream())
    for b, (k, v) in enumerate(dense):
        r = _ref_attn(qd[b:b + 1], k, v, torch.tensor([ctxs[b] - 1], device="cuda"), scale)
        assert rel(od[b:b + 1], r) < 1e-2, b


@pytest.mark.parametrize("qk_norm", [False, True], ids=["llama", "qwen3-qknorm"])
@pytest.mark.parametrize("d_head", [64, 128])
def test_rope_commit(lib, qk_norm, d_head):
    shape = ModelShape("t", 1, 512, 8, 2, d_head, 64, 64, rope_theta=10000.0, rms_eps=1e-6, qk_norm=qk_norm)
    pool = _pool(lib, shape)
    n = 37
    pool.reserve(0, 200)
    pool.sync(torch.cuda.current_stream().cuda_stream)
    qkv = torch.randn(n, (shape.n_q + 2 * shape.n_kv) * shape.d_head, device="cuda") * 3.0
    pos = torch.arange(150, 150 + n, dtype=torch.int32, device="cuda")
    slot_of = torch.zeros(n, dtype=torch.int32, device="cuda")
    q = torch.empty(n, shape.q_dim, dtype=torch.bfloat16, device="cuda")
    qn = (1.0 + 0.1 * torch.randn(d_head, device="cuda")).to(torch.bfloat16)
    kn = (1.0 + 0.1 * torch.randn(d_head, device="cuda")).to(torch.bfloat16)
    qkv0 = qkv.clone()
    if qk_norm:
        lib.call("stb_qkv_norm_rope_commit", pool.h, 0, P(qkv), P(q), P(slot_of), P(pos), n, shape.n_q,
                 shape.rope_theta, P(qn), P(kn), shape.rms_eps, 20, stream())
    else:
        lib.call("stb_qkv_rope_commit", pool.h, 0, P(qkv), P(q), P(slot_of), P(pos), n, shape.n_q,
                 shape.rope_theta, 20, stream())
    assert not qkv[:20].any() and torch.equal(qkv[20:], qkv0[20:])  # consumer clears rows < clear_rows
    qkv = qkv0
    from oracle.cpu_decoder import CpuDecoder

    dec = CpuDecoder.__new__(CpuDecoder)
    dec.s = shape
    dec.inv_freq = torch.tensor([1.0 / math.pow(shape.rope_theta, 2.0 * i / shape.d_head)
                                 for i in range(shape.d_head // 2)], dtype=torch.float32)
    x = qkv.cpu().view(n, -1, shape.d_head)
    xq, xk = x[:, :shape.n_q], x[:, shape.n_q:shape.n_q + shape.n_kv]
    w = {"qn": qn.float().cpu(), "kn": kn.float().cpu()} if qk_norm else {}
    xq, xk = dec._qk(w, xq, xk)
    rq, rk = dec._rope(xq, pos.cpu()), dec._rope(xk, pos.cpu())
    assert rel(q.view(n, shape.n_q, -1).cpu(), rq) < 5e-3
    kd, vd = _dense_kv(pool, 0, 0, 150 + n, shape)
    assert rel(kd[150:].cpu(), rk) < 5e-3
    assert rel(vd[150:].cpu(), x[:, shape.n_q + shape.n_kv:]) < 5e-3


def test_small_ops(lib):
    n, d, f, V = 13, 512, 256, 1000
    ids = torch.randint(0, V, (n,), dtype=torch.int32, device="cuda")
    table = torch.randn(V, d, device="cuda").to(torch.bfloat16)
    x = torch.empty(n, d, device="cuda")
    lib.call("stb_embed", P(ids), P(table), P(x), n, d, stream())
    assert torch.equal(x, table[ids.long()].float())
    delta = torch.randn(n, d, device="cuda")
    w = (1 + 0.1 * torch.randn(d, device="cuda")).to(torch.bfloat16)
    y = torch.empty(n, d, dtype=torch.bfloat16, device="cuda")
    x0 = x.clone()
    delta0 = delta.clone()
    lib.call("stb_add_rmsnorm", P(x), P(delta), P(w), P(y), n, d, 1e-5, n, stream())
    assert not delta.any()
    xr = x0 + delta0
    ref = xr * torch.rsqrt((xr * xr).mean(-1, keepdim=True) + 1e-5) * w.float()
    assert torch.allclose(x, xr) and rel(y, ref) < 5e-3
    gu = torch.randn(n, 2 * f, device="cuda")
    a = torch.empty(n, f, dtype=torch.bfloat16, device="cuda")
    gu0 = gu.clone()
    gate, up = gu0[:, 0::2], gu0[:, 1::2]  # (gate_i, up_i) interleaved
    lib.call("stb_silu_mul", P(gu), P(a), n, f, 0, stream())
    assert rel(a, torch.nn.functional.silu(gate) * up) < 5e-3
    lib.call("stb_silu_mul", P(gu), P(a), n, f, 5, stream())
    assert not gu[:5].any() and torch.equal(gu[5:], gu0[5:])
    assert rel(a, torch.nn.functional.silu(gate) * up) < 5e-3
    idx = torch.tensor([3, 0, 12], dtype=torch.int32, device="cuda")
    rows = torch.empty(3, d, dtype=torch.bfloat16, device="cuda")
    lib.call("stb_gather_rmsnorm", P(x), P(idx), P(w), P(rows), 3, d, 1e-5, stream())
    assert rel(rows, ref[idx.long()]) < 5e-3


def test_sample_forced(lib):
    R, V = 9, 128256
    logits = torch.randn(R, V, device="cuda")
    target = torch.tensor([5, -1, 77, 128255, 0, -1, 3, 9, 1000], dtype=torch.int32, device="cuda")
    out = torch.empty(R, dtype=torch.int32, device="cuda")
    raw = torch.empty(R, dtype=torch.int32, device="cuda")
    mx = torch.empty(R, device="cuda")
    am = logits.argmax(-1).int()
    want = torch.where(target >= 0, target, am)
    top = logits.max(-1).values
    for clear in (0, 1):
        lib.call("stb_sample_forced", P(logits), V, P(target), R, V, 1e4, P(out), P(raw), P(mx), clear, stream())
        assert torch.equal(out, want) and torch.equal(raw, am)
        assert torch.equal(mx, top)
    assert not logits.any()


def test_spec_validate(lib):
    rng = random.Random(0)
    S = 40
    drafts, models, spans, d_off, m_off = [], [], [], [0], [0]
    for _ in range(S):
        L = rng.randrange(0, 70)
        dr = [rng.randrange(5) for _ in range(L)]
        mo = list(dr)
        if L and rng.random() < 0.7:
            mo[rng.randrange(L)] += 1
        mo += [rng.randrange(5) for _ in range(rng.randrange(0, 3))]
        drafts += dr
        models += mo
        spans.append(rng.randrange(1, 80))
        d_off.append(len(drafts))
        m_off.append(len(models))
    t = lambda v: torch.tensor(v if v else [0], dtype=torch.int32, device="cuda")  # noqa: E731
    acc, con, nl = (torch.empty(S, dtype=torch.int32, device="cuda") for _ in range(3))
    kv = t([100 * i for i in range(S)])
    extra = t([i % 2 for i in range(S)])
    firsts = [rng.choice([-1, 0, 1, 2]) for _ in range(S)]
    keep = [t(drafts), t(d_off), t(models), t(m_off), t(firsts), t(spans)]  # alive until the kernel ran
    lib.call("stb_spec_validate", *(P(x) for x in keep), P(kv), P(extra), S, P(acc), P(con), P(nl), stream())
    for s in range(S):
        dr, mo = drafts[d_off[s]:d_off[s + 1]], models[m_off[s]:m_off[s + 1]]
        if firsts[s] >= 0:
            mo = [firsts[s]] + mo
        n = min(len(dr), len(mo), spans[s])
        a = next((i for i in range(n) if dr[i] != mo[i]), n)
        assert acc[s].item() == a
        assert con[s].item() == (spans[s] if a >= spans[s] else a + 1)
        assert nl[s].item() == 100 * s + a + s % 2


def test_error_paths(lib):
    """C-ABI error convention: negative STB_E* codes with a message, mapped to the reference's
    exception types (capacity -> KVCapacityError, the rest -> KernelError); nothing launches."""
    from paper_2512_15834_b200.errors import KernelError, KVCapacityError, SpectoolError

    a = torch.zeros(8, 100, device="cuda", dtype=torch.bfloat16)
    w = torch.zeros(64, 100, device="cuda", dtype=torch.bfloat16)
    c = torch.zeros(8, 64, device="cuda")
    with pytest.raises(KernelError, match="multiple of 8"):  # K % 8 != 0
        lib.call("stb_gemm_bf16", P(a), 100, P(w), 100, P(c), 64, 8, 64, 100 - 4 + 2, 0, 0, stream())
    shape = ModelShape("t", 1, 256, 6, 2, 64, 64, 64)  # group 3: no decode kernel instance
    pool = _pool(lib, shape, nb=8, slots=2, bps=4)
    with pytest.raises(KVCapacityError):  # 8 blocks of 16 rows cannot hold 200 rows
        pool.reserve(0, 200)
    with pytest.raises(KernelError, match="unsupported"):
        q = torch.zeros(1, 6, 64, device="cuda", dtype=torch.bfloat16)
        pool.reserve(1, 16)
        pool.sync(torch.cuda.current_stream().cuda_stream)
        slots = torch.tensor([1], dtype=torch.int32, device="cuda")
        ctx = torch.tensor([16], dtype=torch.int32, device="cuda")
        ws = torch.zeros(1 << 20, device="cuda")
        lib.call("stb_attn_decode", pool.h, 0, P(q), P(q), P(slots), P(ctx), 1, 6, 0.125, 0, P(ws), stream())
    assert issubclass(KernelError, SpectoolError) and issubclass(KVCapacityError, SpectoolError)


@pytest.mark.parametrize("case", ["decode_c2", "decode_c5", "ingest_c5"])
def test_attention_full_size_invariant(lib, case):
    """Size-independent property at BASELINE sizes (no fp32 reference needed): with every V row
    equal to the same vector u, each attention output row is u whatever the scores — the
    softmax weights of every split, merge and masked tile must sum to one. C2: 32 sequences at
    ctx 4096 (K3); C5: 16 sequences at ctx 33k (K3) and a 2048-token ingest at ctx 34816 (K2)."""
    shape = SHAPES[0]  # Llama-3-8B attention geometry
    ctxs = {"decode_c2": [4096] * 32, "decode_c5": [33000] * 16, "ingest_c5": [34816]}[case]
    pool = _pool(lib, shape, nb=sum(-(-c // 16) for c in ctxs) + 8, slots=len(ctxs), bps=2304)
    for b, c in enumerate(ctxs):
        pool.reserve(b, c)
    pool.sync(torch.cuda.current_stream().cuda_stream)
    g = torch.Generator(device="cuda").manual_seed(11)
    u = torch.randn(shape.n_kv, shape.d_head, device="cuda", generator=g).to(torch.bfloat16)
    for b, c in enumerate(ctxs):
        k = (3.0 * torch.randn(c, shape.kv_dim, device="cuda", generator=g)).to(torch.bfloat16)
        v = u.reshape(1, -1).expand(c, -1).contiguous()
        slot_of = torch.full((c,), b, dtype=torch.int32, device="cuda")
        pos = torch.arange(c, dtype=torch.int32, device="cuda")
        lib.call("stb_kv_commit", pool.h, 0, P(k), P(v), shape.kv_dim, P(slot_of), P(pos), c, stream())
    scale = 1 / math.sqrt(shape.d_head)
    want = u.float().repeat_interleave(shape.n_q // shape.n_kv, dim=0)  # [n_q, d]
    if case == "ingest_c5":
        n = 2048
        q = torch.randn(n, shape.n_q, shape.d_head, device="cuda", generator=g).to(torch.bfloat16)
        out = torch.full_like(q, float("nan"))
        slot0 = torch.zeros(1, dtype=torch.int32, device="cuda")
        qstart = torch.tensor([0, n], dtype=torch.int32, device="cuda")
        ctx0 = torch.tensor(ctxs, dtype=torch.int32, device="cuda")
        lib.call("stb_attn_prefill", pool.h, 0, P(q), P(out), P(slot0), P(qstart), P(ctx0), 1, n, shape.n_q, scale, n,
                 stream())
    else:
        B = len(ctxs)
        q = torch.randn(B, shape.n_q, shape.d_head, device="cuda", generator=g).to(torch.bfloat16)
        out = torch.full_like(q, float("nan"))
        slots = torch.arange(B, dtype=torch.int32, device="cuda")
        ctx = torch.tensor(ctxs, dtype=torch.int32, device="cuda")
        ws = torch.zeros(-(-lib.load().stb_attn_decode_workspace(B, shape.n_q, shape.n_kv, shape.d_head) // 4), device="cuda")
        lib.call("stb_attn_decode", pool.h, 0, P(q), P(out), P(slots), P(ctx), B, shape.n_q, scale, 0, P(ws),
                 stream())
    torch.cuda.synchronize()
    err = (out.float() - want).abs().max().item()
    assert err <= 2e-2 * want.abs().max().item(), err


def test_attn_decode_max_batch_and_empty(lib):
    """K3 at its per-launch maximum (STB_K3_MAXB = 1024 sequences, ragged contexts 1..97, so
    the partition cuts many tiny pairs), one past it (EINVAL, nothing launched), and B = 0
    (a no-op that leaves the output untouched)."""
    from paper_2512_15834_b200.errors import KernelError

    shape = SHAPES[0]
    B = 1024
    rng = random.Random(11)
    ctxs = [rng.randint(1, 97) for _ in range(B)]
    pool = _pool(lib, shape, nb=sum(-(-c // 16) for c in ctxs) + 8, slots=B + 1, bps=16)
    dense = _fill_pool(lib, pool, shape, ctxs, seed=4)
    q = torch.randn(B + 1, shape.n_q, shape.d_head, device="cuda").to(torch.bfloat16)
    out = torch.full_like(q, float("nan"))
    slots = torch.arange(B + 1, dtype=torch.int32, device="cuda")
    ctx = torch.tensor(ctxs + [1], dtype=torch.int32, device="cuda")
    ws = torch.zeros(-(-lib.load().stb_attn_decode_workspace(B + 1, shape.n_q, shape.n_kv, shape.d_head) // 4), device="cuda")
    scale = 1 / math.sqrt(shape.d_head)
    lib.call("stb_attn_decode", pool.h, 0, P(q), P(out), P(slots), P(ctx), B, shape.n_q, scale, 0, P(ws), stream())
    worst = 0.0
    for b, (k, v) in enumerate(dense):
        ref = _ref_attn(q[b:b + 1], k, v, torch.tensor([ctxs[b] - 1], device="cuda"), scale)
        worst = max(worst, rel(out[b:b + 1], ref))
    assert worst < 1e-2
    assert torch.isnan(out[B].float()).all()  # row B is not part of the launch
    with pytest.raises(KernelError, match="at most 1024"):
        lib.call("stb_attn_decode", pool.h, 0, P(q), P(out), P(slots), P(ctx), B + 1, shape.n_q, scale, 0, P(ws),
                 stream())
    keep = out.clone()
    lib.call("stb_attn_decode", pool.h, 0, P(q), P(out), P(slots), P(ctx), 0, shape.n_q, scale, 0, P(ws), stream())
    torch.cuda.synchronize()
    assert torch.equal(out[:B], keep[:B])


def test_attn_prefill_empty_runs(lib):
    """K2 with empty runs between non-empty ones (q_start repeats) and S = 0: empty runs
    launch no work and write nothing, the others match the fp32 reference."""
    shape = SHAPES[0]
    runs = [(0, 40), (37, 300), (0, 5), (1, 129)]
    ctxs = [c for _, c in runs]
    pool = _pool(lib, shape, nb=sum(-(-c // 16) for c in ctxs) + 8, slots=len(runs), bps=64)
    dense = _fill_pool(lib, pool, shape, ctxs, seed=9)
    T = sum(n for n, _ in runs)
    q = torch.randn(T, shape.n_q, shape.d_head, device="cuda").to(torch.bfloat16)
    out = torch.full_like(q, float("nan"))
    qs = [0]
    for n, _ in runs:
        qs.append(qs[-1] + n)
    slots = torch.arange(len(runs), dtype=torch.int32, device="cuda")
    qstart = torch.tensor(qs, dtype=torch.int32, device="cuda")
    ctx = torch.tensor(ctxs, dtype=torch.int32, device="cuda")
    scale = 1 / math.sqrt(shape.d_head)
    lib.call("stb_attn_prefill", pool.h, 0, P(q), P(out), P(slots), P(qstart), P(ctx), len(runs), T, shape.n_q,
             scale, max(n for n, _ in runs), stream())
    for s, ((n, c), (k, v)) in enumerate(zip(runs, dense)):
        if n:
            ref = _ref_attn(q[qs[s]:qs[s + 1]], k, v, torch.arange(c - n, c, device="cuda"), scale)
            assert rel(out[qs[s]:qs[s + 1]], ref) < 1e-2, s
    keep = out.clone()
    lib.call("stb_attn_prefill", pool.h, 0, P(q), P(out), P(slots), P(qstart), P(ctx), 0, T, shape.n_q, scale, 1,
             stream())
    torch.cuda.synchronize()
    assert torch.equal(out, keep)


def test_attn_decode_graph_survives_larger_batch(lib):
    """K3's split-merge tickets live in the caller's workspace, so a CUDA
    graph captured at a small B still replays correctly after an eager launch at a larger B
    (which used to free and reallocate a hidden ticket array under the captured graph), and
    the ticket region is all zero again after every launch."""
    shape = SHAPES[2]  # Qwen3-32B geometry: n_kv 8, the C3 config of the advisor's report
    ctxs_big = [3000 + 37 * i for i in range(40)]
    pool = _pool(lib, shape, nb=sum(-(-c // 16) for c in ctxs_big) + 8, slots=len(ctxs_big), bps=512)
    dense = _fill_pool(lib, pool, shape, ctxs_big, seed=12)
    scale = 1 / math.sqrt(shape.d_head)
    nb = lib.load().stb_attn_decode_workspace(64, shape.n_q, shape.n_kv, shape.d_head)
    ws = torch.zeros(-(-nb // 4), device="cuda")
    Bs = 4
    q = torch.randn(len(ctxs_big), shape.n_q, shape.d_head, device="cuda").to(torch.bfloat16)
    out_s = torch.empty(Bs, shape.n_q, shape.d_head, device="cuda", dtype=torch.bfloat16)
    slots = torch.arange(len(ctxs_big), dtype=torch.int32, device="cuda")
    ctx = torch.tensor(ctxs_big, dtype=torch.int32, device="cuda")
    g = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        lib.call("stb_attn_decode", pool.h, 0, P(q), P(out_s), P(slots), P(ctx), Bs, shape.n_q, scale, 0, P(ws),
                 stream())
    out_b = torch.empty_like(q)
    lib.call("stb_attn_decode", pool.h, 0, P(q), P(out_b), P(slots), P(ctx), len(ctxs_big), shape.n_q, scale, 0,
             P(ws), stream())
    out_s.fill_(float("nan"))
    g.replay()
    torch.cuda.synchronize()
    for b, (k, v) in enumerate(dense):
        r = _ref_attn(q[b:b + 1], k, v, torch.tensor([ctxs_big[b] - 1], device="cuda"), scale)
        assert rel(out_b[b:b + 1], r) < 1e-2, b
        if b < Bs:
            assert rel(out_s[b:b + 1], r) < 1e-2, b
    tickets = ws.view(torch.int32)[-(64 * shape.n_kv + 64):]
    assert int(tickets.abs().sum()) == 0


def test_kv_copy_blocks(lib):
    """K1 fork / copy-on-write: stb_kv_copy_blocks duplicates whole blocks (every layer, K and V);
    the copy's dense view equals the source's, and the source is untouched."""
    shape = ModelShape("t", 3, 256, 4, 2, 64, 64, 64)
    pool = _pool(lib, shape, nb=64, slots=4)
    dense = _fill_pool(lib, pool, shape, [37], seed=3)
    n = 37
    pool.reserve(1, n)  # destination slot: its own 3 blocks
    pool.sync(torch.cuda.current_stream().cuda_stream)
    src = torch.tensor(pool.blocks(0), dtype=torch.int32, device="cuda")
    dst = torch.tensor(pool.blocks(1), dtype=torch.int32, device="cuda")
    assert set(src.tolist()).isdisjoint(dst.tolist())
    lib.call("stb_kv_copy_blocks", pool.h, P(src), P(dst), len(src), stream())
    torch.cuda.synchronize()
    k0, v0 = dense[0]
    for layer in range(shape.layers):
        ks, vs = _dense_kv(pool, layer, 0, n, shape)
        kd, vd = _dense_kv(pool, layer, 1, n, shape)
        assert torch.equal(ks, k0) and torch.equal(vs, v0)
        assert torch.equal(kd, k0) and torch.equal(vd, v0)
    lib.call("stb_kv_copy_blocks", pool.h, P(src), P(dst), 0, stream())  # empty call: no-op
