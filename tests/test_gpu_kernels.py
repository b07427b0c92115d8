"""GPU parity of the compute kernels: tcgen05 GEMM (every tile width and
epilogue), fused add-bias+residual+LayerNorm, fused varlen MHA (short and
long paths) -- against fp32 references (torch fp32 for the GEMM/LN, the
pinned oracle for attention) on the same bf16-rounded inputs."""

import math

import numpy as np
import pytest

from oracle import packbert_np as orc
from tests._metrics import assert_close_bf16, cosine, rel_fro

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch

    import paper_2210_03052_b200 as bt

    bt._lib.require_device()
    torch.manual_seed(0)
    return bt, torch


@pytest.fixture
def two_cta_mha(env):
    """The two-CTAs-per-SM MHA kernels (mha_sm100.cu) for the packed launches
    the four-CTA kernel (mha64_sm100.cu) serves by default: their scheduling
    modes are pinned bitwise against each other and against the oracle."""
    from paper_2210_03052_b200 import _lib

    _lib.call("bt_debug_mha64", 0)
    yield
    _lib.call("bt_debug_mha64", -1)


def _gelu(t):
    return 0.5 * t * (1.0 + torch_tanh(math.sqrt(2 / math.pi) * (t + 0.044715 * t ** 3)))


def torch_tanh(t):
    import torch

    return torch.tanh(t)


@pytest.mark.parametrize("bn", [64, 128, 192, 256, -112, -128, -176, -192, -224, -240, -256])
@pytest.mark.parametrize("epi", [0, 1, 2, 3])
@pytest.mark.parametrize("M,N,K", [(1, 768, 64), (200, 768, 768), (2458, 2304, 768), (129, 1024, 4096),
                                   (300, 3072, 128)])
def test_gemm(env, bn, epi, M, N, K):
    bt, torch = env
    from paper_2210_03052_b200.tensor import gemm_device

    # N % BN != 0 (e.g. N = 1024 with 192-wide tiles) runs a partial last N
    # tile: B rows past N zero-filled by TMA, columns past N never stored
    a = (torch.randn(M, K, device="cuda") * 0.5).to(torch.bfloat16)
    w = (torch.randn(N, K, device="cuda") / math.sqrt(K)).to(torch.bfloat16)
    bias = torch.randn(N, device="cuda") * 0.1
    res = torch.randn(M, N, device="cuda").to(torch.bfloat16)
    out = gemm_device(a, w, bias if epi else None, res if epi == 3 else None, epi, bn=bn)
    ref = a.float() @ w.float().t()
    if epi == 3:
        ref = ref + res.float()
    if epi:
        ref = ref + bias
    if epi == 2:
        ref = _gelu(ref)
    torch.cuda.synchronize()
    assert rel_fro(out, ref) < 6e-3, (bn, epi, M, N, K, rel_fro(out, ref))
    assert (out.float() - ref).abs().max().item() < 0.05 * max(1.0, ref.abs().max().item())


def test_gemm_public_api(env):
    bt, torch = env
    rng = np.random.default_rng(1)
    a = rng.standard_normal((37, 128)).astype(np.float32)
    b = (rng.standard_normal((128, 192)) * 0.1).astype(np.float32)
    bias = rng.standard_normal(192).astype(np.float32)
    got = bt.gemm(bt.Tensor(a), bt.Tensor(b), bt.EpilogueHook.add_bias_gelu(bias))
    ref = orc.gelu(a @ b + bias)
    assert_close_bf16(got, ref, rel_max=1e-2, what="gemm+bias+gelu")
    q, k, v = bt.batched_gemm([bt.Tensor(a)] * 3, [bt.Tensor(b[:, :64]), bt.Tensor(b[:, 64:128]),
                                                    bt.Tensor(b[:, 128:])])
    assert_close_bf16(k, a @ b[:, 64:128], rel_max=1e-2, what="batched")
    with pytest.raises(bt.ShapeError):
        bt.gemm(bt.Tensor(a), bt.Tensor(b[:64]))


@pytest.mark.parametrize("K,N", [(100, 50), (7, 3), (64, 130)])
def test_gemm_public_api_any_shape(env, K, N):
    """The reference gemm takes any shape (tensor.py:177-200); K and N that
    are not multiples of 64 run zero-padded on the device."""
    bt, torch = env
    rng = np.random.default_rng(K * 1000 + N)
    a = rng.standard_normal((45, K)).astype(np.float32)
    b = (rng.standard_normal((K, N)) * 0.1).astype(np.float32)
    bias = rng.standard_normal(N).astype(np.float32)
    got = bt.gemm(bt.Tensor(a), bt.Tensor(b), bt.EpilogueHook.add_bias(bias))
    assert got.array.shape == (45, N)
    assert_close_bf16(got, a @ b + bias, rel_max=1e-2, what=f"gemm {K}x{N}")
    got = bt.gemm(bt.Tensor(a), bt.Tensor(b))
    assert_close_bf16(got, a @ b, rel_max=1e-2, what=f"gemm {K}x{N} no epilogue")


@pytest.mark.parametrize("k", [768, 1024, 64, 2048])
def test_layernorm(env, k):
    bt, torch = env
    from paper_2210_03052_b200.fusion import ln_device

    T = 1000
    x = torch.randn(T, k, device="cuda").to(torch.bfloat16)
    r = torch.randn(T, k, device="cuda").to(torch.bfloat16)
    b = torch.randn(k, device="cuda") * 0.1
    g = torch.randn(k, device="cuda")
    be = torch.randn(k, device="cuda")
    out = ln_device(x, r, b, g, be, 1e-12)
    z = (x.float() + r.float()) + b
    ref = torch.nn.functional.layer_norm(z, (k,), g, be, eps=1e-12)
    assert rel_fro(out, ref) < 5e-3
    # constant rows normalise to exactly beta (variance 0, reference fusion.py:52-53)
    c = torch.full((4, k), 3.0, device="cuda").to(torch.bfloat16)
    outc = ln_device(c, None, None, g, be, 1e-12)
    assert torch.allclose(outc.float(), be.to(torch.bfloat16).float().expand(4, k), atol=1e-2)


def test_layernorm_golden(env, golden):
    bt, torch = env
    g = golden("fusion")
    y = bt.add_bias_residual_layernorm(bt.Tensor(g["ln_x"]), bt.Tensor(g["ln_r"]), g["ln_b"],
                                       bt.LayernormParams(g["ln_g"], g["ln_beta"]))
    assert_close_bf16(y, g["ln_y"], what="LN vs reference")
    kat = bt.layernorm(bt.Tensor(np.array([[1, 2, 3, 0, 0, 0, 0, 0]], np.float32)),
                       bt.LayernormParams(np.ones(8, np.float32), np.zeros(8, np.float32)))
    ref = orc.layernorm(np.array([[1, 2, 3, 0, 0, 0, 0, 0]], np.float32), np.ones(8), np.zeros(8))
    assert np.abs(kat.array - ref).max() < 2e-2


def test_gelu_and_elementwise(env, golden):
    bt, torch = env
    g = golden("fusion")
    got = bt.gelu(g["gelu_in"])
    assert np.abs(got - g["gelu_out"]).max() < 2e-2  # bf16-free fp32 path, tanh.approx
    assert abs(float(bt.gelu(np.float32(1.0))) - 0.841192) < 2e-3
    a = np.random.default_rng(0).standard_normal((5, 16)).astype(np.float32)
    np.testing.assert_allclose(bt.add(bt.Tensor(a), bt.Tensor(a)).array, 2 * a, rtol=1e-6)
    np.testing.assert_allclose(bt.add_rowvec(bt.Tensor(a), np.ones(16, np.float32)).array, a + 1, rtol=1e-6)


def _attn_case(golden, tag):
    g = golden("attention")
    lens = g[f"{tag}_lengths"].tolist()
    mx, heads = int(g[f"{tag}_mx"]), int(g[f"{tag}_heads"])
    return g, lens, mx, heads


@pytest.mark.parametrize("tag", ["short", "long", "cut384", "cut385"])
def test_mha_golden(env, golden, tag):
    """dispatch_mha on the reference's own attention vectors."""
    bt, torch = env
    g, lens, mx, heads = _attn_case(golden, tag)
    plan = bt.plan_for_lengths(bt.SeqLengths.of(lens, mx))
    hid = heads * 64
    b = g[f"{tag}_bias"]
    inp = bt.AttentionInput(bt.Tensor(g[f"{tag}_q"]), bt.Tensor(g[f"{tag}_k"]), bt.Tensor(g[f"{tag}_v"]),
                            b[:hid], b[hid:2 * hid], b[2 * hid:], plan, heads, 64)
    out = bt.dispatch_mha(inp)
    assert_close_bf16(out, g[f"{tag}_out"], what=f"mha {tag}")


def _rand_qkv(torch, T, hid, scale=1.0, seed=0):
    gen = torch.Generator(device="cuda").manual_seed(seed)
    return (torch.randn(T, 3 * hid, device="cuda", generator=gen) * scale).to(torch.bfloat16)


def _oracle_mha(qkv, plan, heads, mx, cutoff=384):
    a = qkv.float().cpu().numpy()
    hid = heads * 64
    zero = np.zeros(3 * hid, np.float32)
    return orc.dispatch_mha(a[:, :hid], a[:, hid:2 * hid], a[:, 2 * hid:], zero, plan.seq_starts, mx, heads, 64,
                            cutoff)


@pytest.mark.parametrize("mha64", [1, 0])
@pytest.mark.parametrize("path", [1, 2])
@pytest.mark.parametrize("lens,mx", [([1, 2, 3, 127, 128, 129, 200, 256], 256), ([384, 1, 383, 257, 77], 384),
                                     ([5] * 40, 8), ([128] * 6, 128), ([64, 63, 65, 1, 191, 193], 200)])
def test_mha_paths_random(env, path, lens, mx, mha64):
    """Every kernel on edge lengths (1, the 64- and 128-key block boundaries,
    384) with N(0,1) q/k/v (sharp softmax), vs the fp32 oracle: the
    four-CTA kernel (mha64 = 1, 64-key blocks) and the two-CTA resident
    (path 1) / streamed (path 2) kernels."""
    bt, torch = env
    from paper_2210_03052_b200 import _lib
    from paper_2210_03052_b200.attention import mha_device

    heads = 3
    plan = bt.plan_for_lengths(bt.SeqLengths.of(lens, mx))
    qkv = _rand_qkv(torch, plan.valid_word_cnt, heads * 64, seed=len(lens))
    _lib.call("bt_debug_mha64", mha64)
    try:
        out = mha_device(qkv, plan, heads, 64, path=path)
    finally:
        _lib.call("bt_debug_mha64", -1)
    ref = _oracle_mha(qkv, plan, heads, mx)
    assert_close_bf16(out, ref, what=f"mha64={mha64} path{path} {lens[:4]}")


@pytest.mark.parametrize("lens,mx", [([1000, 1, 513, 640, 129], 1024), ([512] * 3 + [300], 512)])
def test_mha_long_random(env, lens, mx):
    bt, torch = env
    from paper_2210_03052_b200.attention import mha_device

    heads = 2
    plan = bt.plan_for_lengths(bt.SeqLengths.of(lens, mx))
    qkv = _rand_qkv(torch, plan.valid_word_cnt, heads * 64, seed=7)
    out = mha_device(qkv, plan, heads, 64)
    ref = _oracle_mha(qkv, plan, heads, mx)
    assert_close_bf16(out, ref, what="long")


def test_mha_padded_token_isolation(env):
    """Tokens of other sequences never influence a sequence: perturbing
    sequence 1 leaves sequences 0 and 2 bitwise unchanged."""
    bt, torch = env
    from paper_2210_03052_b200.attention import mha_device

    for mx in (256, 700):
        lens = [100, 150, 60] if mx == 256 else [600, 300, 700]
        plan = bt.plan_for_lengths(bt.SeqLengths.of(lens, mx))
        qkv = _rand_qkv(torch, plan.valid_word_cnt, 128, seed=3)
        a = mha_device(qkv, plan, 2, 64).clone()
        s = plan.seq_starts
        qkv2 = qkv.clone()
        qkv2[s[1]:s[2]] = torch.randn_like(qkv2[s[1]:s[2]].float()).to(torch.bfloat16) * 5
        b = mha_device(qkv2, plan, 2, 64)
        assert torch.equal(a[: s[1]], b[: s[1]]) and torch.equal(a[s[2]:], b[s[2]:])


def test_mha_deterministic(env):
    bt, torch = env
    from paper_2210_03052_b200.attention import mha_device

    plan = bt.plan_for_lengths(bt.SeqLengths.of([300, 17, 256], 512))
    qkv = _rand_qkv(torch, plan.valid_word_cnt, 256, seed=9)
    a = mha_device(qkv, plan, 4, 64).clone()
    b = mha_device(qkv, plan, 4, 64)
    assert torch.equal(a, b)


@pytest.mark.parametrize("bn", [64, 128, 256, -128, -192, -256])
@pytest.mark.parametrize("epi", [0, 2, 3])
@pytest.mark.parametrize("M,N,K", [(2458, 768, 3072), (2458, 2304, 768), (300, 768, 128), (77, 768, 64),
                                   (4915, 1024, 4096)])
def test_gemm_streamk(env, bn, epi, M, N, K):
    """Stream-K decomposition (forced on): split tiles are fixed up from fp32
    partials in a fixed order -- results match the fp32 reference and are
    bitwise reproducible run to run."""
    bt, torch = env
    from paper_2210_03052_b200 import _lib
    from paper_2210_03052_b200.tensor import gemm_device

    if N % abs(bn):
        pytest.skip("N not a multiple of BN")
    a = (torch.randn(M, K, device="cuda") * 0.5).to(torch.bfloat16)
    w = (torch.randn(N, K, device="cuda") / math.sqrt(K)).to(torch.bfloat16)
    bias = torch.randn(N, device="cuda") * 0.1
    res = torch.randn(M, N, device="cuda").to(torch.bfloat16)
    _lib.call("bt_debug_gemm_mode", 4)
    try:
        out = gemm_device(a, w, bias if epi else None, res if epi == 3 else None, epi, bn=bn)
        out2 = gemm_device(a, w, bias if epi else None, res if epi == 3 else None, epi, bn=bn)
    finally:
        _lib.call("bt_debug_gemm_mode", 5)
    ref = a.float() @ w.float().t()
    if epi == 3:
        ref = ref + res.float()
    if epi:
        ref = ref + bias
    if epi == 2:
        ref = _gelu(ref)
    torch.cuda.synchronize()
    assert rel_fro(out, ref) < 6e-3, (bn, epi, M, N, K, rel_fro(out, ref))
    assert torch.equal(out, out2)


@pytest.mark.parametrize("path,lens,mx", [(1, [384, 300, 140, 129], 384), (2, [700, 260, 131], 768)])
def test_mha_reference_max_moves(env, path, lens, mx):
    """Keys 128..255 of every sequence get 4x larger logits, so a row's max
    jumps by more than 2^8 in P units after the first key block: the
    kernel's lazily moved reference max must rescale O and l in place."""
    bt, torch = env
    from paper_2210_03052_b200.attention import mha_device

    heads = 2
    hid = heads * 64
    plan = bt.plan_for_lengths(bt.SeqLengths.of(lens, mx))
    qkv = _rand_qkv(torch, plan.valid_word_cnt, hid, seed=11)
    s = plan.seq_starts
    for b in range(len(lens)):
        lo, hi = s[b] + 128, min(s[b] + 256, s[b + 1])
        if hi > lo:
            qkv[lo:hi, hid:2 * hid] *= 4  # exact in bf16
    out = mha_device(qkv, plan, heads, 64, path=path)
    ref = _oracle_mha(qkv, plan, heads, mx)
    assert_close_bf16(out, ref, what=f"rescale path{path}")


@pytest.mark.parametrize("M,N,K", [(2458, 768, 768), (2458, 768, 3072), (1, 768, 64), (300, 1024, 1024),
                                   (129, 512, 256), (4915, 1024, 4096)])
def test_gemm_bias_residual_ln(env, M, N, K):
    """Fused projection + add-bias + residual + LayerNorm (one cluster of N/128
    CTAs per 128-row block, row statistics over DSMEM) vs torch fp32 of
    LN((A W^T + R) + b) on the same bf16 operands."""
    bt, torch = env
    from paper_2210_03052_b200.fusion import gemm_ln_device

    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    A = (torch.randn(M, K, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    W = (torch.randn(N, K, device="cuda", generator=g) / math.sqrt(K)).to(torch.bfloat16)
    R = (torch.randn(M, N, device="cuda", generator=g) * 2 + 0.5).to(torch.bfloat16)
    b = torch.randn(N, device="cuda", generator=g) * 0.1
    gamma = 1 + torch.randn(N, device="cuda", generator=g) * 0.1
    beta = torch.randn(N, device="cuda", generator=g) * 0.1
    out = gemm_ln_device(A, W, b, R, gamma, beta, 1e-12)
    z = (A.float() @ W.float().t() + R.float()) + b
    ref = torch.nn.functional.layer_norm(z, (N,), gamma, beta, eps=1e-12)
    assert_close_bf16(out, ref, what=f"gemm_ln {M}x{N}x{K}")


def test_mha_sched_order_is_result_neutral(env):
    """The longest-first CTA schedule (bt_plan_sched) changes only the
    dispatch order: outputs are bitwise those of the natural order, and the
    schedule lists every sequence once, by descending key-block count."""
    bt, torch = env
    from paper_2210_03052_b200 import _lib
    from paper_2210_03052_b200.attention import mha_device

    lens = [5, 300, 129, 1, 512, 128, 257, 77]
    mx, H = 512, 2
    plan = bt.plan_for_lengths(bt.SeqLengths.of(lens, mx))
    T = plan.valid_word_cnt
    qkv = _rand_qkv(torch, T, H * 64, seed=5)
    nbytes = _lib.load().bt_plan_sched_bytes(len(lens), mx)
    sched = torch.zeros(nbytes // 4, dtype=torch.int32, device="cuda")
    _lib.call("bt_plan_sched", plan.seq_starts_dev.data_ptr(), len(lens), mx, sched.data_ptr(), _lib.stream_ptr())
    out = torch.empty(T, H * 64, device="cuda", dtype=torch.bfloat16)
    _lib.call("bt_mha_varlen_sched", qkv.data_ptr(), plan.seq_starts_dev.data_ptr(), sched.data_ptr(), len(lens), mx,
              H, 64, 384, out.data_ptr(), T, _lib.stream_ptr())
    ref = mha_device(qkv, plan, H, 64)
    assert torch.equal(out, ref)
    pairs = sched[:2 * len(lens)].view(-1, 2).cpu().numpy()
    starts = plan.seq_starts
    assert sorted(map(tuple, pairs)) == sorted((int(starts[b]), lens[b]) for b in range(len(lens)))
    blocks = [(l + 127) // 128 for _, l in pairs]
    assert blocks == sorted(blocks, reverse=True)


@pytest.mark.parametrize("grid", [0, 1, 3, 7, 64])
@pytest.mark.parametrize("lens,mx", [([5, 300, 129, 1, 512, 128, 257, 77], 512), ([256, 140, 9, 255, 1, 2], 256),
                                     ([1000, 3, 700, 129], 1024)])
def test_mha_tile_list(env, two_cta_mha, lens, mx, grid):
    """The tile-list MHA (a fixed grid claims bt_plan_sched's query tiles x
    heads longest-first from a queue; what the forward runs for launches of
    many waves) is bitwise the one-tile-per-CTA kernel,
    for any grid size -- one CTA walking everything, fewer CTAs than heads,
    more CTAs than items -- and the unit list covers every query tile once,
    longest sequences first."""
    bt, torch = env
    from paper_2210_03052_b200 import _lib
    from paper_2210_03052_b200.attention import mha_device

    H = 3
    plan = bt.plan_for_lengths(bt.SeqLengths.of(lens, mx))
    T = plan.valid_word_cnt
    qkv = _rand_qkv(torch, T, H * 64, seed=11)
    nbytes = _lib.load().bt_plan_sched_bytes(len(lens), mx)
    sched = torch.full((nbytes // 4,), -1, dtype=torch.int32, device="cuda")
    _lib.call("bt_plan_sched", plan.seq_starts_dev.data_ptr(), len(lens), mx, sched.data_ptr(), _lib.stream_ptr())
    out = torch.full((T, H * 64), float("nan"), device="cuda", dtype=torch.bfloat16)
    _lib.call("bt_debug_mha_list", 2, grid)
    _lib.call("bt_debug_mha_seg", 0)
    try:
        _lib.call("bt_mha_varlen_sched", qkv.data_ptr(), plan.seq_starts_dev.data_ptr(), sched.data_ptr(), len(lens),
                  mx, H, 64, 384, out.data_ptr(), T, _lib.stream_ptr())
    finally:
        _lib.call("bt_debug_mha_list", -1, 0)
        _lib.call("bt_debug_mha_seg", -1)
    torch.cuda.synchronize()
    ref = mha_device(qkv, plan, H, 64)
    assert torch.equal(out, ref)
    # unit list: every (sequence, query tile) once, descending key blocks
    off = (2 * len(lens) * 4 + 15) // 16 * 4
    n = int(sched[off].item())
    units = sched[off + 4: off + 4 + 2 * n].view(-1, 2).cpu().numpy()
    starts = plan.seq_starts
    want = sorted((int(starts[b]), q, lens[b]) for b in range(len(lens)) for q in range((lens[b] + 127) // 128))
    got = sorted((int(s0), int(w) >> 20, int(w) & 0xFFFFF) for s0, w in units)
    assert got == want
    blocks = [((int(w) & 0xFFFFF) + 127) // 128 for _, w in units]
    assert blocks == sorted(blocks, reverse=True)


@pytest.mark.parametrize("lens,mx", [([512, 300, 129, 1, 450, 257], 512), ([256, 140, 9, 255], 256),
                                     ([1000, 3, 700], 1024)])
def test_mha_query_tiles_per_cta(env, two_cta_mha, lens, mx):
    """The multi-tile MHA variant (a CTA walks several query tiles of its
    sequence-head; chosen automatically for launches of many waves) is bitwise
    the single-tile kernel, which the other tests pin to the oracle."""
    bt, torch = env
    from paper_2210_03052_b200 import _lib
    from paper_2210_03052_b200.attention import mha_device

    plan = bt.plan_for_lengths(bt.SeqLengths.of(lens, mx))
    qkv = _rand_qkv(torch, plan.valid_word_cnt, 2 * 64, seed=13)
    try:
        _lib.call("bt_debug_mha_qg", 1)
        one = mha_device(qkv, plan, 2, 64).clone()
        for qg in (2, 4, 8):
            _lib.call("bt_debug_mha_qg", qg)
            assert torch.equal(mha_device(qkv, plan, 2, 64), one), f"qg={qg}"
    finally:
        _lib.call("bt_debug_mha_qg", 0)


def _mha_sched_call(bt, torch, qkv, plan, heads, mx, cutoff=384):
    from paper_2210_03052_b200 import _lib

    bs = plan.batch_size
    T = plan.valid_word_cnt
    sched = torch.full((_lib.load().bt_plan_sched_bytes(bs, mx) // 4,), -1, dtype=torch.int32, device="cuda")
    _lib.call("bt_plan_sched", plan.seq_starts_dev.data_ptr(), bs, mx, sched.data_ptr(), _lib.stream_ptr())
    out = torch.full((T, heads * 64), float("nan"), device="cuda", dtype=torch.bfloat16)
    _lib.call("bt_mha_varlen_sched", qkv.data_ptr(), plan.seq_starts_dev.data_ptr(), sched.data_ptr(), bs, mx, heads,
              64, cutoff, out.data_ptr(), T, _lib.stream_ptr())
    torch.cuda.synchronize()
    return out


@pytest.mark.parametrize("lens,mx", [([1, 2, 3, 127, 128, 129, 200, 256], 256), ([5] * 40, 8),
                                     ([1] * 250 + [64, 250], 256), ([100, 28, 128, 1, 127, 129, 60], 256),
                                     ([244, 190, 157, 96, 105, 36, 45, 30, 70, 234, 192, 256, 154, 181, 256, 212], 256),
                                     ([64] * 200, 64)])
def test_mha_segment_kernel(env, lens, mx):
    """The segment kernel (query tiles of sequences > 128 rows, and groups of
    adjacent short sequences sharing one 128-row tile with each row masked
    to its own sequence -- what the forward runs for bs, max_seq_len <= 256)
    vs the fp32 oracle: groups of hundreds of 1-token sequences, exact
    128-row groups, the C2 batch."""
    bt, torch = env
    from paper_2210_03052_b200 import _lib

    heads = 3
    plan = bt.plan_for_lengths(bt.SeqLengths.of(lens, mx))
    qkv = _rand_qkv(torch, plan.valid_word_cnt, heads * 64, seed=len(lens) + 3)
    _lib.call("bt_debug_mha_seg", 2)
    try:
        out = _mha_sched_call(bt, torch, qkv, plan, heads, mx)
    finally:
        _lib.call("bt_debug_mha_seg", -1)
    assert torch.isfinite(out.float()).all()
    ref = _oracle_mha(qkv, plan, heads, mx)
    assert_close_bf16(out, ref, what=f"segments {lens[:4]}")


def test_mha_segment_kernel_isolation_and_rescale(env):
    """Segment kernel: a sequence's output does not depend on its window
    neighbours (perturbing every other sequence's q/k/v leaves it bitwise
    unchanged), and a late jump of the row max (keys 128.. scaled 4x) is
    rescaled correctly."""
    bt, torch = env
    from paper_2210_03052_b200 import _lib

    lens, mx, heads = [37, 200, 5, 256, 90, 1, 140], 256, 2
    hid = heads * 64
    plan = bt.plan_for_lengths(bt.SeqLengths.of(lens, mx))
    qkv = _rand_qkv(torch, plan.valid_word_cnt, hid, seed=21)
    s = plan.seq_starts
    for b in range(len(lens)):
        lo, hi = s[b] + 128, min(s[b] + 256, s[b + 1])
        if hi > lo:
            qkv[lo:hi, hid:2 * hid] *= 4
    _lib.call("bt_debug_mha_seg", 2)
    try:
        out = _mha_sched_call(bt, torch, qkv, plan, heads, mx)
        ref = _oracle_mha(qkv, plan, heads, mx)
        assert_close_bf16(out, ref, what="segments rescale")
        pert = qkv.clone()
        for b in range(len(lens)):
            if b != 1:
                pert[s[b]:s[b + 1]] = (torch.randn_like(pert[s[b]:s[b + 1]].float()) * 3).to(torch.bfloat16)
        out2 = _mha_sched_call(bt, torch, pert, plan, heads, mx)
    finally:
        _lib.call("bt_debug_mha_seg", -1)
    assert torch.equal(out[s[1]:s[2]], out2[s[1]:s[2]])
