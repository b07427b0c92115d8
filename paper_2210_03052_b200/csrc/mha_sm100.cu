// Fused variable-length multi-head attention on tcgen05 (paper section III-E,
// reference attention.py:177-314).  Both kernels index the packed [T, 3k]
// QKV tensor through seq_starts and never touch a padded token.
//
// One CTA = (q-tile of 128 rows, head, sequence); 4 warps, thread t owns
// query row t of the tile == TMEM lane t, so row max / row sum are
// thread-local (no shuffles) and the softmax reads S straight out of TMEM.
//
//   short path (max_seq_len <= cutoff, attention.py:177-237): the whole
//     K/V head slab of the sequence (<= 384 keys) is TMA-staged in shared
//     memory once, S = Q K^T for every key lands in TMEM (<= 384 fp32
//     columns), the exact row softmax is taken over the full row (no
//     rescaling, as the reference's tile-local softmax), P (bf16) is written
//     to shared memory in the UMMA K-major 128B-swizzled layout and
//     O = P V accumulates in TMEM.
//   long path (max_seq_len > cutoff, attention.py:240-296): keys are streamed
//     in 128-key blocks through a 2-deep TMA ring; the reference's
//     "partial (max, sum) per 128-column tile + full reduction + exp on load"
//     is carried out as the equivalent single-pass online softmax (per-block
//     partial max/sum merged into running statistics), so P never goes to
//     HBM.  Work per CTA is sized by the sequence's true length (grouped
//     problem sizes).
//
// Q/K/V biases are already applied by the QKV GEMM epilogue.  d = 64.

#include "common.cuh"
#include "ptx.cuh"
#include "tma_host.cuh"

namespace bt {

constexpr int MHA_D = 64;
constexpr int MHA_QT = 128;                  // query rows per CTA (UMMA M)
constexpr int MHA_KB = 128;                  // keys per block (UMMA N of S)
constexpr uint32_t MHA_TILE = 128 * 128;     // bytes of one 128 x 64 bf16 tile
constexpr int MHA_SHORT_MAX_KEYS = 384;      // TMEM: 384 S columns + 64 O columns <= 512

struct MhaParams {
  const int32_t* seq_starts;
  __nv_bfloat16* out;
  int hidden;      // H * d
  float sl2;       // softmax scale * log2(e)
};

// Write 32 consecutive bf16 P values (packed in 16 u32) of row `row`,
// starting at key column `c` (multiple of 32), into the K-major SW128 layout:
// 64-key column blocks of 128 rows x 128 B, 16 B chunks XOR-swizzled by row%8.
__device__ __forceinline__ void store_p32(uint8_t* sP, int row, int c, const uint32_t (&pk)[16]) {
  uint8_t* blk = sP + (c >> 6) * MHA_TILE + row * 128;
  const int chunk0 = (c & 63) >> 3;
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int phys = (chunk0 + t) ^ (row & 7);
    *reinterpret_cast<uint4*>(blk + phys * 16) = make_uint4(pk[4 * t], pk[4 * t + 1], pk[4 * t + 2], pk[4 * t + 3]);
  }
}

__device__ __forceinline__ void store_out_row(const MhaParams& p, int grow, int h, const float (&o)[64], float inv) {
  uint4* dst = reinterpret_cast<uint4*>(p.out + static_cast<size_t>(grow) * p.hidden + h * MHA_D);
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    uint4 v;
    v.x = ptx::pack_bf16x2(o[8 * q + 0] * inv, o[8 * q + 1] * inv);
    v.y = ptx::pack_bf16x2(o[8 * q + 2] * inv, o[8 * q + 3] * inv);
    v.z = ptx::pack_bf16x2(o[8 * q + 4] * inv, o[8 * q + 5] * inv);
    v.w = ptx::pack_bf16x2(o[8 * q + 6] * inv, o[8 * q + 7] * inv);
    dst[q] = v;
  }
}

// ============================================================ short path
template <int NKB>
struct ShortCfg {
  static constexpr uint32_t Q_OFF = 0;
  static constexpr uint32_t K_OFF = MHA_TILE;
  static constexpr uint32_t V_OFF = K_OFF + NKB * MHA_TILE;
  static constexpr uint32_t P_OFF = V_OFF + NKB * MHA_TILE;
  static constexpr uint32_t BAR_OFF = P_OFF + NKB * 2 * MHA_TILE;
  static constexpr size_t SMEM = 1024 + BAR_OFF + 64;
};

template <int NKB>
__global__ void __launch_bounds__(128, 1) mha_short_kernel(const __grid_constant__ CUtensorMap tm, const MhaParams p) {
  using Cfg = ShortCfg<NKB>;
  const int qt = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int s0 = __ldg(p.seq_starts + b);
  const int len = __ldg(p.seq_starts + b + 1) - s0;
  const int q0 = qt * MHA_QT;
  if (q0 >= len) return;  // CTA-uniform: this q tile is past the sequence
  const int nkb = (len + MHA_KB - 1) / MHA_KB;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem + Cfg::Q_OFF;
  uint8_t* sK = smem + Cfg::K_OFF;
  uint8_t* sV = smem + Cfg::V_OFF;
  uint8_t* sP = smem + Cfg::P_OFF;
  uint64_t* ld_bar = reinterpret_cast<uint64_t*>(smem + Cfg::BAR_OFF);
  uint64_t* mma_bar = ld_bar + 1;
  uint32_t* holder = reinterpret_cast<uint32_t*>(ld_bar + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    ptx::prefetch_tmap(&tm);
    ptx::mbar_init(ld_bar, 1);
    ptx::mbar_init(mma_bar, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 0) {
    ptx::tmem_alloc(holder, 512);
    ptx::tmem_relinquish();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *holder;
  constexpr uint32_t O_COL = MHA_SHORT_MAX_KEYS;
  ptx::griddep_launch_dependents();
  ptx::griddep_wait();  // qkv is produced by the previous kernel

  if (threadIdx.x == 0) {
    // stage Q tile and the whole K/V head slab of this sequence
    ptx::mbar_arrive_expect_tx(ld_bar, (1 + 2 * nkb) * MHA_TILE);
    ptx::tma_load_2d(sQ, &tm, ld_bar, h * MHA_D, s0 + q0);
    for (int j = 0; j < nkb; ++j) {
      ptx::tma_load_2d(sK + j * MHA_TILE, &tm, ld_bar, p.hidden + h * MHA_D, s0 + j * MHA_KB);
      ptx::tma_load_2d(sV + j * MHA_TILE, &tm, ld_bar, 2 * p.hidden + h * MHA_D, s0 + j * MHA_KB);
    }
    ptx::mbar_wait(ld_bar, 0);
    ptx::tc_fence_after();
    constexpr uint32_t idesc_s = ptx::idesc_bf16(128, 128, false, false);
    const uint32_t q_addr = ptx::smem_u32(sQ);
    for (int j = 0; j < nkb; ++j) {
      const uint32_t k_addr = ptx::smem_u32(sK + j * MHA_TILE);
#pragma unroll
      for (int kk = 0; kk < MHA_D / 16; ++kk)
        ptx::mma_bf16_ss(tmem + j * MHA_KB, ptx::sdesc_sw128(q_addr + kk * 32, 1024, 16),
                         ptx::sdesc_sw128(k_addr + kk * 32, 1024, 16), idesc_s, kk > 0);
    }
    ptx::mma_commit(mma_bar);
  }
  __syncwarp();
  ptx::mbar_wait(mma_bar, 0);
  ptx::tc_fence_after();

  // ---- exact row softmax straight out of TMEM (thread = row)
  const int row = warp * 32 + lane;
  const uint32_t trow = tmem + (static_cast<uint32_t>(warp * 32) << 16);
  const int kcols = nkb * MHA_KB;
  float mrow = -INFINITY;
  for (int c = 0; c < kcols; c += 32) {
    uint32_t r[32];
    ptx::tmem_ld32(trow + c, r);
    ptx::tmem_wait_ld(r);
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (c + i < len) mrow = fmaxf(mrow, __uint_as_float(r[i]));
  }
  const float msc = mrow * p.sl2;
  float lsum = 0.f;
  for (int c = 0; c < kcols; c += 32) {
    uint32_t r[32];
    ptx::tmem_ld32(trow + c, r);
    ptx::tmem_wait_ld(r);
    uint32_t pk[16];
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
      const float e0 = (c + i < len) ? ptx::ex2_approx(fmaf(__uint_as_float(r[i]), p.sl2, -msc)) : 0.f;
      const float e1 = (c + i + 1 < len) ? ptx::ex2_approx(fmaf(__uint_as_float(r[i + 1]), p.sl2, -msc)) : 0.f;
      lsum += e0 + e1;
      pk[i / 2] = ptx::pack_bf16x2(e0, e1);
    }
    store_p32(sP, row, c, pk);
  }
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();

  if (threadIdx.x == 0) {
    constexpr uint32_t idesc_o = ptx::idesc_bf16(128, MHA_D, false, true);  // P K-major, V MN-major
    const uint32_t p_addr = ptx::smem_u32(sP);
    const uint32_t v_addr = ptx::smem_u32(sV);
    const int nks = (len + 15) / 16;
    for (int ks = 0; ks < nks; ++ks) {
      const uint64_t ad = ptx::sdesc_sw128(p_addr + (ks >> 2) * MHA_TILE + (ks & 3) * 32, 1024, 16);
      const uint64_t bd = ptx::sdesc_sw128(v_addr + ks * 16 * 128, 1024, MHA_TILE);
      ptx::mma_bf16_ss(tmem + O_COL, ad, bd, idesc_o, ks > 0);
    }
    ptx::mma_commit(mma_bar);
  }
  __syncwarp();
  ptx::mbar_wait(mma_bar, 1);
  ptx::tc_fence_after();
  float o[64];
  {
    uint32_t r[32];
    ptx::tmem_ld32(trow + O_COL, r);
    ptx::tmem_wait_ld(r);
#pragma unroll
    for (int i = 0; i < 32; ++i) o[i] = __uint_as_float(r[i]);
    ptx::tmem_ld32(trow + O_COL + 32, r);
    ptx::tmem_wait_ld(r);
#pragma unroll
    for (int i = 0; i < 32; ++i) o[32 + i] = __uint_as_float(r[i]);
  }
  if (q0 + row < len) store_out_row(p, s0 + q0 + row, h, o, 1.0f / lsum);

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

// ============================================================ long path
struct LongCfg {
  static constexpr uint32_t Q_OFF = 0;
  static constexpr uint32_t K_OFF = MHA_TILE;          // 2 stages
  static constexpr uint32_t V_OFF = K_OFF + 2 * MHA_TILE;
  static constexpr uint32_t P_OFF = V_OFF + 2 * MHA_TILE;  // 128 keys = 2 column blocks
  static constexpr uint32_t BAR_OFF = P_OFF + 2 * MHA_TILE;
  static constexpr size_t SMEM = 1024 + BAR_OFF + 64;
};

__global__ void __launch_bounds__(128, 1) mha_long_kernel(const __grid_constant__ CUtensorMap tm, const MhaParams p) {
  using Cfg = LongCfg;
  const int qt = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int s0 = __ldg(p.seq_starts + b);
  const int len = __ldg(p.seq_starts + b + 1) - s0;
  const int q0 = qt * MHA_QT;
  if (q0 >= len) return;
  const int nkb = (len + MHA_KB - 1) / MHA_KB;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem + Cfg::Q_OFF;
  uint8_t* sK = smem + Cfg::K_OFF;
  uint8_t* sV = smem + Cfg::V_OFF;
  uint8_t* sP = smem + Cfg::P_OFF;
  uint64_t* kv_full = reinterpret_cast<uint64_t*>(smem + Cfg::BAR_OFF);  // [2]
  uint64_t* s_bar = kv_full + 2;
  uint64_t* pv_bar = kv_full + 3;
  uint32_t* holder = reinterpret_cast<uint32_t*>(kv_full + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    ptx::prefetch_tmap(&tm);
    ptx::mbar_init(&kv_full[0], 1);
    ptx::mbar_init(&kv_full[1], 1);
    ptx::mbar_init(s_bar, 1);
    ptx::mbar_init(pv_bar, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 0) {
    ptx::tmem_alloc(holder, 256);
    ptx::tmem_relinquish();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *holder;
  constexpr uint32_t S_COL = 0, O_COL = 128;
  ptx::griddep_launch_dependents();
  ptx::griddep_wait();  // qkv is produced by the previous kernel
  constexpr uint32_t idesc_s = ptx::idesc_bf16(128, 128, false, false);
  constexpr uint32_t idesc_o = ptx::idesc_bf16(128, MHA_D, false, true);

  if (threadIdx.x == 0) {
    ptx::mbar_arrive_expect_tx(&kv_full[0], 3 * MHA_TILE);
    ptx::tma_load_2d(sQ, &tm, &kv_full[0], h * MHA_D, s0 + q0);
    ptx::tma_load_2d(sK, &tm, &kv_full[0], p.hidden + h * MHA_D, s0);
    ptx::tma_load_2d(sV, &tm, &kv_full[0], 2 * p.hidden + h * MHA_D, s0);
    if (nkb > 1) {
      ptx::mbar_arrive_expect_tx(&kv_full[1], 2 * MHA_TILE);
      ptx::tma_load_2d(sK + MHA_TILE, &tm, &kv_full[1], p.hidden + h * MHA_D, s0 + MHA_KB);
      ptx::tma_load_2d(sV + MHA_TILE, &tm, &kv_full[1], 2 * p.hidden + h * MHA_D, s0 + MHA_KB);
    }
  }

  const int row = warp * 32 + lane;
  const uint32_t trow = tmem + (static_cast<uint32_t>(warp * 32) << 16);
  float o[64];
#pragma unroll
  for (int i = 0; i < 64; ++i) o[i] = 0.f;
  float mrow = -INFINITY, lsum = 0.f;
  const uint32_t q_addr = ptx::smem_u32(sQ);
  const uint32_t p_addr = ptx::smem_u32(sP);

  for (int j = 0; j < nkb; ++j) {
    const int st = j & 1;
    const uint32_t par = j & 1;
    if (threadIdx.x == 0) {
      ptx::mbar_wait(&kv_full[st], (j >> 1) & 1);
      ptx::tc_fence_after();
      const uint32_t k_addr = ptx::smem_u32(sK + st * MHA_TILE);
#pragma unroll
      for (int kk = 0; kk < MHA_D / 16; ++kk)
        ptx::mma_bf16_ss(tmem + S_COL, ptx::sdesc_sw128(q_addr + kk * 32, 1024, 16),
                         ptx::sdesc_sw128(k_addr + kk * 32, 1024, 16), idesc_s, kk > 0);
      ptx::mma_commit(s_bar);
    }
    __syncwarp();
    ptx::mbar_wait(s_bar, par);
    ptx::tc_fence_after();

    // per-block partial max (reference: per-128-column tile partials,
    // tensor.py:166-173) merged into the running row statistics
    const int kbase = j * MHA_KB;
    float bmax = -INFINITY;
    for (int c = 0; c < MHA_KB; c += 32) {
      uint32_t r[32];
      ptx::tmem_ld32(trow + S_COL + c, r);
      ptx::tmem_wait_ld(r);
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (kbase + c + i < len) bmax = fmaxf(bmax, __uint_as_float(r[i]));
    }
    const float mnew = fmaxf(mrow, bmax);
    const float alpha = ptx::ex2_approx((mrow - mnew) * p.sl2);  // 0 on the first block
    const float msc = mnew * p.sl2;
    float bsum = 0.f;
    for (int c = 0; c < MHA_KB; c += 32) {
      uint32_t r[32];
      ptx::tmem_ld32(trow + S_COL + c, r);
      ptx::tmem_wait_ld(r);
      uint32_t pk[16];
#pragma unroll
      for (int i = 0; i < 32; i += 2) {
        const float e0 =
            (kbase + c + i < len) ? ptx::ex2_approx(fmaf(__uint_as_float(r[i]), p.sl2, -msc)) : 0.f;
        const float e1 =
            (kbase + c + i + 1 < len) ? ptx::ex2_approx(fmaf(__uint_as_float(r[i + 1]), p.sl2, -msc)) : 0.f;
        bsum += e0 + e1;
        pk[i / 2] = ptx::pack_bf16x2(e0, e1);
      }
      store_p32(sP, row, c, pk);
    }
    lsum = lsum * alpha + bsum;
    mrow = mnew;
#pragma unroll
    for (int i = 0; i < 64; ++i) o[i] *= alpha;

    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (threadIdx.x == 0) {
      const uint32_t v_addr = ptx::smem_u32(sV + st * MHA_TILE);
      const int nks = min(MHA_KB, len - kbase + 15) / 16;
      for (int ks = 0; ks < nks; ++ks) {
        const uint64_t ad = ptx::sdesc_sw128(p_addr + (ks >> 2) * MHA_TILE + (ks & 3) * 32, 1024, 16);
        const uint64_t bd = ptx::sdesc_sw128(v_addr + ks * 16 * 128, 1024, MHA_TILE);
        ptx::mma_bf16_ss(tmem + O_COL, ad, bd, idesc_o, ks > 0);
      }
      ptx::mma_commit(pv_bar);
    }
    __syncwarp();
    ptx::mbar_wait(pv_bar, par);
    ptx::tc_fence_after();
    {
      uint32_t r[32];
      ptx::tmem_ld32(trow + O_COL, r);
      ptx::tmem_wait_ld(r);
#pragma unroll
      for (int i = 0; i < 32; ++i) o[i] += __uint_as_float(r[i]);
      ptx::tmem_ld32(trow + O_COL + 32, r);
      ptx::tmem_wait_ld(r);
#pragma unroll
      for (int i = 0; i < 32; ++i) o[32 + i] += __uint_as_float(r[i]);
    }
    // stage st is free (its S and PV MMAs retired): prefetch block j + 2
    if (threadIdx.x == 0 && j + 2 < nkb) {
      ptx::mbar_arrive_expect_tx(&kv_full[st], 2 * MHA_TILE);
      ptx::tma_load_2d(sK + st * MHA_TILE, &tm, &kv_full[st], p.hidden + h * MHA_D, s0 + (j + 2) * MHA_KB);
      ptx::tma_load_2d(sV + st * MHA_TILE, &tm, &kv_full[st], 2 * p.hidden + h * MHA_D, s0 + (j + 2) * MHA_KB);
    }
    ptx::tc_fence_before();
    __syncthreads();  // S / O_part TMEM and sP are reused by the next block
    ptx::tc_fence_after();
  }
  if (q0 + row < len) store_out_row(p, s0 + q0 + row, h, o, 1.0f / lsum);

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 256);
  }
}

template <typename K>
static int set_smem(K kern, size_t bytes) {
  BT_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
  return BT_OK;
}

int mha_launch(const void* qkv, const int32_t* seq_starts, int bs, int mx, int H, int d, int cutoff, int T,
               void* out, int force_path, cudaStream_t s) {
  BT_REQUIRE(d == MHA_D, BT_ECONFIG, "fused MHA supports head_size 64, got %d", d);
  BT_REQUIRE(bs >= 1 && mx >= 1 && H >= 1 && T >= 1, BT_ESHAPE, "mha: bad shape bs=%d mx=%d H=%d T=%d", bs, mx, H, T);
  const int hidden = H * d;
  CUtensorMap tm;
  BT_TRY(make_tmap_bf16_2d(&tm, qkv, T, 3 * hidden, 3 * hidden, 128, 64));
  MhaParams p;
  p.seq_starts = seq_starts;
  p.out = static_cast<__nv_bfloat16*>(out);
  p.hidden = hidden;
  p.sl2 = 1.4426950408889634f / sqrtf(static_cast<float>(d));
  const dim3 grid((mx + MHA_QT - 1) / MHA_QT, H, bs);
  // dispatch_mha rule (attention.py:309-314); the on-chip short kernel holds
  // at most 384 keys.
  bool use_short = mx <= cutoff && mx <= MHA_SHORT_MAX_KEYS;
  if (force_path == 1) use_short = true;
  if (force_path == 2) use_short = false;
  BT_REQUIRE(!use_short || mx <= MHA_SHORT_MAX_KEYS, BT_ECONFIG, "short MHA holds <= 384 keys, mx=%d", mx);
  if (use_short) {
    const int nkb = (mx + MHA_KB - 1) / MHA_KB;
    static bool set1 = false, set2 = false, set3 = false;
    if (nkb == 1) {
      if (!set1) { BT_TRY(set_smem(mha_short_kernel<1>, ShortCfg<1>::SMEM)); set1 = true; }
      BT_LAUNCH(mha_short_kernel<1>, grid, dim3(128), ShortCfg<1>::SMEM, s, 1, tm, p);
    } else if (nkb == 2) {
      if (!set2) { BT_TRY(set_smem(mha_short_kernel<2>, ShortCfg<2>::SMEM)); set2 = true; }
      BT_LAUNCH(mha_short_kernel<2>, grid, dim3(128), ShortCfg<2>::SMEM, s, 1, tm, p);
    } else {
      if (!set3) { BT_TRY(set_smem(mha_short_kernel<3>, ShortCfg<3>::SMEM)); set3 = true; }
      BT_LAUNCH(mha_short_kernel<3>, grid, dim3(128), ShortCfg<3>::SMEM, s, 1, tm, p);
    }
  } else {
    static bool setl = false;
    if (!setl) { BT_TRY(set_smem(mha_long_kernel, LongCfg::SMEM)); setl = true; }
    BT_LAUNCH(mha_long_kernel, grid, dim3(128), LongCfg::SMEM, s, 1, tm, p);
  }
  return BT_OK;
}

}  // namespace bt

extern "C" int bt_mha_varlen(const void* qkv, const int32_t* seq_starts, int bs, int mx, int H, int d, int cutoff,
                             int split_seq_len, void* out, int T, bt_stream_t stream) {
  BT_REQUIRE(split_seq_len >= 1, BT_ESHAPE, "split_seq_len must be >= 1, got %d", split_seq_len);
  return bt::mha_launch(qkv, seq_starts, bs, mx, H, d, cutoff, T, out, 0, bt::as_stream(stream));
}

// Test hook: force the short (1) or long (2) kernel regardless of cutoff.
extern "C" int bt_mha_varlen_path(const void* qkv, const int32_t* seq_starts, int bs, int mx, int H, int d,
                                  void* out, int T, int path, bt_stream_t stream) {
  return bt::mha_launch(qkv, seq_starts, bs, mx, H, d, 384, T, out, path, bt::as_stream(stream));
}
