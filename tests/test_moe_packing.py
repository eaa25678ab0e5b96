"""MoE expert packing on the CPU (no GPU): the MX stage layout the block-scaled grouped GEMM
(csrc/moe.cu moe_gemm_mx_kernel) reads — one 3-D TMA box of packed codes plus the scale words in
the tcgen05.cp [lane][column] layout — checked element by element against the codes / exponents."""

import torch

from paper_2512_15834_b200.runtime import weights as W


def test_pack_mx_stages():
    """MX stage layout: codes row-major in 64-byte rows, scale word (l, j) = row 32 j + l."""
    N, K = 200, 320
    g = torch.Generator().manual_seed(3)
    codes = torch.randint(0, 16, (N, K), generator=g).to(torch.uint8)
    exps = torch.randint(-13, 13, (N, K // 32), generator=g).to(torch.int8)
    st = W.pack_mx_stages(codes, exps)
    assert st.shape == (2, 3, W.MX_STAGE_BYTES)
    for n, r, s_, k in [(0, 0, 0, 0), (1, 71, 2, 63), (0, 127, 1, 100), (1, 50, 0, 5)]:
        row = n * 128 + r
        b = int(st[n, s_, r * 64 + k // 2])
        kk = s_ * 128 + k
        want = int(codes[row, kk]) if row < N and kk < K else 0
        assert (b >> (4 * (k & 1))) & 15 == want
        word = st[n, s_, 8192:].view(torch.int32)[(r % 32) * 4 + r // 32].item() & 0xFFFFFFFF
        for t in range(4):
            blk = s_ * 4 + t
            want_s = int(exps[row, blk]) + 127 if row < N and blk < K // 32 else 127
            assert (word >> (8 * t)) & 255 == want_s


def test_pack_mx_stages_roundtrip():
    """Every code and scale byte lands where the kernel reads it (full unpack vs the inputs)."""
    N, K = 130, 192
    g = torch.Generator().manual_seed(5)
    codes = torch.randint(0, 16, (N, K), generator=g).to(torch.uint8)
    exps = torch.randint(-13, 13, (N, K // 32), generator=g).to(torch.int8)
    st = W.pack_mx_stages(codes, exps)
    NT, KS = st.shape[:2]
    b = st[..., :8192].reshape(NT, KS, 128, 64)
    full = torch.stack([b & 15, b >> 4], -1).reshape(NT, KS, 128, 128).permute(0, 2, 1, 3).reshape(NT * 128, KS * 128)
    assert torch.equal(full[:N, :K], codes) and not full[N:].any() and not full[:, K:].any()
    w = st[..., 8192:].reshape(NT, KS, 32, 4, 4)  # [n][s][lane][column j][byte t] = row 32 j + lane
    sc = w.permute(0, 3, 2, 1, 4).reshape(NT * 128, KS * 4).to(torch.int16) - 127
    assert torch.equal(sc[:N, :K // 32], exps.to(torch.int16))
    assert not sc[:, K // 32:].any() and not sc[N:].any()
