"""Probe: GPU kernels reading / writing page-locked host memory directly
(UVA zero-copy) vs DMA copies, for the e2e input / output of C2."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    import paper_2210_03052_b200 as bt
    from paper_2210_03052_b200 import _lib, harness

    _lib.require_device()
    bs, mx, k = 16, 256, 768
    seqs = harness.gen_lengths(bs, mx, "fixed", seed=0, alpha=0.6)
    plan = bt.plan_for_lengths(seqs)
    T = plan.valid_word_cnt
    xh = torch.from_numpy(harness.gen_input(seqs, k, 0)).pin_memory()
    yh = torch.empty((bs * mx, k), dtype=torch.float32).pin_memory()
    xd = torch.empty((bs * mx, k), dtype=torch.float32, device="cuda")
    packed = torch.empty((T, k), dtype=torch.bfloat16, device="cuda")
    s = torch.cuda.current_stream()

    def timeit(fn, n=20):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(n):
            fn()
        b.record(s)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / n * 1e3

    nbytes = T * k * 4
    zc_in = timeit(lambda: _lib.call("bt_pack_starts", xh.data_ptr(), plan.seq_starts_dev.data_ptr(), bs, mx, k,
                                     packed.data_ptr(), _lib.stream_ptr()))
    dma_in = timeit(lambda: xd.copy_(xh, non_blocking=True))
    zc_out = timeit(lambda: _lib.call("bt_unpack", packed.data_ptr(), _lib.BT_BF16, plan.seq_starts_dev.data_ptr(), bs,
                                      mx, k, yh.data_ptr(), _lib.BT_F32, _lib.stream_ptr()))
    dma_out = timeit(lambda: yh.copy_(xd, non_blocking=True))
    print(f"zero-copy gather of {nbytes / 1e6:.1f} MB valid fp32 rows from host: {zc_in:.1f} us "
          f"({nbytes / zc_in / 1e3:.1f} GB/s)")
    print(f"DMA of the whole padded input ({xh.numel() * 4 / 1e6:.1f} MB): {dma_in:.1f} us "
          f"({xh.numel() * 4 / dma_in / 1e3:.1f} GB/s)")
    print(f"zero-copy scatter to host padded fp32 (incl. zero rows, {yh.numel() * 4 / 1e6:.1f} MB): {zc_out:.1f} us "
          f"({yh.numel() * 4 / zc_out / 1e3:.1f} GB/s)")
    print(f"DMA of the whole padded output: {dma_out:.1f} us ({yh.numel() * 4 / dma_out / 1e3:.1f} GB/s)")
    ref = bt.pack_device(xh.cuda(), plan, out_dtype=torch.bfloat16) if hasattr(bt, "pack_device") else None
    from paper_2210_03052_b200.packing import pack_device
    _lib.call("bt_pack_starts", xh.data_ptr(), plan.seq_starts_dev.data_ptr(), bs, mx, k, packed.data_ptr(),
              _lib.stream_ptr())
    torch.cuda.synchronize()
    print("zero-copy gather matches device pack:", torch.equal(packed, pack_device(xh.cuda(), plan,
                                                                                    out_dtype=torch.bfloat16)))


if __name__ == "__main__":
    main()
