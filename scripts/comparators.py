"""Same-box comparators: the fused varlen MHA against
flash_attn.flash_attn_varlen_func and flashinfer's ragged prefill, and the
layer GEMMs against cuBLAS (torch.matmul, bf16), on C2 / C3 / C5 shapes.
Library kernels are context here, not the bar (the reference has no GPU
path).  CUDA-event timing, back-to-back launches after warm-up, L2-warm.

    python scripts/comparators.py [--out profiles/r01_comparators.json]
"""

import argparse
import json
import math
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

CONFIGS = {"c2": (16, 256, 12, 768), "c3": (16, 512, 16, 1024), "c5": (2048, 512, 16, 1024)}


def timed(torch, fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # ~10 ms of device sleep first: the host enqueues every rep meanwhile, so
    # per-call host overhead (ctypes, torch dispatch) stays out of the timing
    torch.cuda._sleep(int(2e7))
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3  # us


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--configs", nargs="+", default=["c2", "c3", "c5"])
    a = ap.parse_args()
    import torch

    from paper_2210_03052_b200 import _lib, harness
    from paper_2210_03052_b200.packing import plan_for_lengths
    from paper_2210_03052_b200.tensor import gemm_device

    _lib.require_device()
    L = _lib.load()
    res = {"note": "us per launch, CUDA events over back-to-back launches after warm-up, L2-warm inputs; "
                   "MHA FLOPs 4*sum(len^2)*k", "configs": {}}
    for name in a.configs:
        bs, mx, H, k = CONFIGS[name]
        reps = 3 if name == "c5" else 50
        seqs = harness.gen_lengths(bs, mx, "fixed", seed=0, alpha=0.6)
        plan = plan_for_lengths(seqs)
        T = plan.valid_word_cnt
        flops = 4.0 * sum(n * n for n in seqs.lengths) * k
        gen = torch.Generator(device="cuda").manual_seed(0)
        qkv = torch.randn(T, 3 * k, device="cuda", generator=gen).to(torch.bfloat16)
        out = torch.empty(T, k, device="cuda", dtype=torch.bfloat16)
        sched = torch.zeros(L.bt_plan_sched_bytes(bs, mx) // 4 + 1, dtype=torch.int32, device="cuda")
        _lib.call("bt_plan_sched", plan.seq_starts_dev.data_ptr(), bs, mx, sched.data_ptr(), _lib.stream_ptr())
        row = {"T": T, "sum_len2": int(sum(n * n for n in seqs.lengths)), "mha": {}, "gemm": {}}

        def ours():
            _lib.call("bt_mha_varlen_sched", qkv.data_ptr(), plan.seq_starts_dev.data_ptr(), sched.data_ptr(), bs, mx,
                      H, 64, 384, out.data_ptr(), T, _lib.stream_ptr())

        us = timed(torch, ours, reps)
        row["mha"]["bt200"] = {"us": round(us, 2), "tflops": round(flops / us / 1e6, 1)}
        q = qkv[:, :k].view(T, H, 64)
        kk = qkv[:, k:2 * k].view(T, H, 64)
        v = qkv[:, 2 * k:].view(T, H, 64)
        cu = plan.seq_starts_dev.to(torch.int32)
        try:
            from flash_attn import flash_attn_varlen_func

            def fa():
                return flash_attn_varlen_func(q, kk, v, cu, cu, mx, mx, softmax_scale=1 / 8.0, causal=False)

            us = timed(torch, fa, reps)
            ref = fa().reshape(T, k)
            row["mha"]["flash_attn_varlen"] = {"us": round(us, 2), "tflops": round(flops / us / 1e6, 1),
                                               "max_abs_diff_vs_bt200": float((ref.float() - out.float()).abs().max())}
        except Exception as e:  # noqa: BLE001
            row["mha"]["flash_attn_varlen"] = {"error": f"{type(e).__name__}: {str(e)[:160]}"}
        try:
            import flashinfer

            ws = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
            w = flashinfer.prefill.BatchPrefillWithRaggedKVCacheWrapper(ws, "NHD")
            w.plan(cu, cu, H, H, 64, causal=False, q_data_type=torch.bfloat16, kv_data_type=torch.bfloat16)

            def fi():
                return w.run(q, kk, v)

            us = timed(torch, fi, reps)
            ref = fi().reshape(T, k)
            row["mha"]["flashinfer_ragged_prefill"] = {
                "us": round(us, 2), "tflops": round(flops / us / 1e6, 1),
                "max_abs_diff_vs_bt200": float((ref.float() - out.float()).abs().max())}
        except Exception as e:  # noqa: BLE001
            row["mha"]["flashinfer_ragged_prefill"] = {"error": f"{type(e).__name__}: {str(e)[:160]}"}
        # layer GEMMs: ours (with the forward's epilogue) vs cuBLAS bf16 (no epilogue)
        x = torch.randn(T, k, device="cuda", generator=gen).to(torch.bfloat16)
        h = torch.randn(T, 4 * k, device="cuda", generator=gen).to(torch.bfloat16)
        for gname, A, N, epi in (("qkv", x, 3 * k, _lib.EPI_BIAS), ("attn_out", x, k, _lib.EPI_NONE),
                                 ("ffn1_gelu", x, 4 * k, _lib.EPI_BIAS_GELU), ("ffn2", h, k, _lib.EPI_NONE)):
            K = A.shape[1]
            W = (torch.randn(N, K, device="cuda", generator=gen) / math.sqrt(K)).to(torch.bfloat16)
            bias = torch.zeros(N, device="cuda")
            C = torch.empty(T, N, device="cuda", dtype=torch.bfloat16)
            gf = 2.0 * T * N * K
            u1 = timed(torch, lambda: gemm_device(A, W, bias if epi else None, None, epi, out=C), reps)
            Wt = W.t()
            u2 = timed(torch, lambda: torch.matmul(A, Wt), reps)
            # cuBLASLt with the same epilogue fused (bias / bias + tanh-GELU)
            b16 = bias.to(torch.bfloat16)
            if epi == _lib.EPI_BIAS:
                u3 = timed(torch, lambda: torch.addmm(b16, A, Wt), reps)
            elif epi == _lib.EPI_BIAS_GELU:
                u3 = timed(torch, lambda: torch._addmm_activation(b16, A, Wt, use_gelu=True), reps)
            else:
                u3 = u2
            row["gemm"][gname] = {"M": T, "N": N, "K": K, "bt200_us": round(u1, 2),
                                  "bt200_tflops": round(gf / u1 / 1e6, 1), "cublas_us": round(u2, 2),
                                  "cublas_tflops": round(gf / u2 / 1e6, 1), "cublas_same_epilogue_us": round(u3, 2)}
        res["configs"][name] = row
        print(name, json.dumps(row), flush=True)
    if a.out:
        Path(a.out).write_text(json.dumps(res, indent=1) + "\n")


if __name__ == "__main__":
    main()
