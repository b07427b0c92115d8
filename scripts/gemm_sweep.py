"""Time every GEMM tile variant on the encoder's shapes (and cuBLAS for
context), checking each result against torch fp32.

    python scripts/gemm_sweep.py [--shapes c2|c3|big|all]
"""

import argparse
import json
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

SHAPES = {
    "c2": [(2458, 2304, 768, 1), (2458, 768, 768, 0), (2458, 3072, 768, 2), (2458, 768, 3072, 0)],
    "c3": [(4915, 3072, 1024, 1), (4915, 1024, 1024, 0), (4915, 4096, 1024, 2), (4915, 1024, 4096, 0)],
    "big": [(78643, 3072, 1024, 1), (78643, 4096, 1024, 2), (78643, 1024, 4096, 0), (8192, 8192, 8192, 0)],
}
VARIANTS = [None, 64, 128, 192, 256, -112, -128, -176, -192, -224, -240, -256]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="all")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--mode", type=int, default=0, help="bt_debug_gemm_mode (0 normal, 1 no-MMA, 2 no-TMA)")
    ap.add_argument("--sk", type=int, default=-1, help="stream-K: -1 auto, 0 off, 1 on")
    a = ap.parse_args()
    import torch

    from paper_2210_03052_b200 import _lib
    from paper_2210_03052_b200.tensor import gemm_device

    _lib.require_device()
    _lib.call("bt_debug_gemm_mode", a.mode)
    _lib.call("bt_debug_gemm_mode", {-1: 5, 0: 3, 1: 4}[a.sk])
    peak = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())["bf16_tflops"]
    groups = list(SHAPES) if a.shapes == "all" else [a.shapes]
    out = []
    for g in groups:
        for (M, N, K, epi) in SHAPES[g]:
            A = (torch.randn(M, K, device="cuda") * 0.5).to(torch.bfloat16)
            W = (torch.randn(N, K, device="cuda") / math.sqrt(K)).to(torch.bfloat16)
            bias = torch.randn(N, device="cuda") * 0.1
            C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
            ref = None
            if M * N <= 2e8:
                ref = A.float() @ W.float().t()
                if epi:
                    ref = ref + bias
                if epi == 2:
                    ref = 0.5 * ref * (1 + torch.tanh(math.sqrt(2 / math.pi) * (ref + 0.044715 * ref ** 3)))
            flops = 2.0 * M * N * K
            row = {"shape": [M, N, K], "epi": epi, "mode": a.mode, "sk": a.sk}
            for v in VARIANTS + (["cublas"] if a.mode == 0 else []):
                if isinstance(v, int) and (N % 64 or 4 * (-(-N // abs(v)) * abs(v) - N) > N):
                    continue  # the partial-last-tile rule of the library's autotuner
                if v == "cublas":
                    fn = lambda: torch.matmul(A, W.t(), out=C)  # noqa: E731
                else:
                    fn = lambda v=v: gemm_device(A, W, bias if epi else None, None, epi, out=C, bn=v)  # noqa: E731
                try:
                    fn()
                    torch.cuda.synchronize()
                except Exception as e:  # noqa: BLE001
                    row[str(v)] = f"ERR {e}"
                    continue
                err = None
                if ref is not None and v != "cublas" and a.mode == 0:
                    err = float((C.float() - ref).norm() / ref.norm())
                ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda._sleep(int(3e7))
                ev0.record()
                for _ in range(a.reps):
                    fn()
                ev1.record()
                torch.cuda.synchronize()
                us = ev0.elapsed_time(ev1) * 1e3 / a.reps
                tf = flops / us / 1e6
                row[str(v)] = {"us": round(us, 2), "tflops": round(tf, 1), "frac": round(tf / peak, 3),
                               "relerr": None if err is None else round(err, 5)}
            out.append(row)
            print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
