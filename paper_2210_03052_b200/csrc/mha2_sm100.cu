// Fused variable-length multi-head attention, persistent form (paper
// section III-E; reference attention.py:177-314, dispatch_mha's two paths in
// one kernel).  What the encoder forward runs.
//
// Work items (bt_plan_sched's segment list, longest problems first): a
// 128-row query tile of one sequence with that sequence's keys, or -- small
// batches -- a group of adjacent short sequences whose rows fit one tile,
// each row masked to its own sequence.  Units = items x heads.  A fixed grid
// of two CTAs per SM claims units from a device queue, one unit ahead of the
// one it computes, so the next unit's Q load and first Q K^T overlap the
// current unit's last softmax block and output store; the per-unit fixed cost
// that a one-tile-per-CTA launch pays in full (Q load ~0.4 us, first S ~0.5 us,
// epilogue ~0.6 us, CTA turnover) is hidden behind the softmax.
//
// Per CTA (256 threads, two per SM):
//   warps 0-3   softmax + epilogue, thread = query row = TMEM lane: a row's
//               128 scores of a key block are in one thread's registers (no
//               cross-thread row max), P goes to TMEM as bf16 (the A operand
//               of O += P V), O / l -> bf16 -> smem -> coalesced 16 B stores
//   warp 4      TMA producer: unit claims, Q (double-buffered), K / V ring
//   warp 5      tcgen05.mma issuer (elect.sync): S = Q K^T, O += P V
//   warps 6-7   idle (complete warpgroup 1 for setmaxnreg)
// TMEM (256 columns): S [0,128) fp32, P [128,192) bf16 pairs, O [192,256).
// Softmax: single pass with a lazily moved reference max (it moves only when
// the block max exceeds it by 2^8 in P units, then O and the row sum are
// rescaled), P = 2^((s - m_ref) * scale * log2 e), two of every sixteen
// exponentials as a polynomial on the FMA pipe.  O / l is exact for any
// reference point: the reference long path's per-tile (max, sum) partials
// with a full reduction (tensor.py:166-173, grouped.py:202-206) without P
// ever leaving the SM.

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "ptx.cuh"
#include "tma_host.cuh"

namespace bt {

constexpr int M2_D = 64;
constexpr int M2_BLK = 128;                  // keys per block = query rows per tile
constexpr uint32_t M2_TILE = 128 * 128;      // bytes of one 128 x 64 bf16 tile
constexpr int M2_THREADS = 256;
constexpr int M2_REGS_SOFTMAX = 200;         // 128 x 200 + 128 x 56 = 32768: two CTAs per SM
constexpr int M2_REGS_ISSUE = 56;
constexpr float M2_RESCALE_LOG2 = 8.0f;
#ifndef BT_MHA2_POLY
#define BT_MHA2_POLY 2  // of every 16 exponentials, this many run as ex2_poly2 on the FMA pipe
#endif

struct M2Smem {
  static constexpr uint32_t Q_OFF = 0;                       // 2 x 16 KB (double-buffered Q)
  static constexpr uint32_t KV_OFF = 2 * M2_TILE;            // 2 slots x (K 16 KB, V 16 KB)
  static constexpr uint32_t OUT_OFF = KV_OFF + 4 * M2_TILE;  // 16 KB output staging
  static constexpr uint32_t BAR_OFF = OUT_OFF + M2_TILE;
  static constexpr size_t SMEM = BAR_OFF + 256;
};

struct Mha2Params {
  __nv_bfloat16* out;
  const int32_t* seq_starts;
  const int4* items;  // 2 int4 per item: {kv start, kv end, q start, q end}, {seq a, seq b, -, -}
  const int* header;  // [0] items, [1] claim queue (next unit), [2] finished CTAs
  int* queue;         // = header + 1
  int hidden;
  int heads;
  float sl2;
  unsigned long long* flops;  // optional instrumented FlopCounter ("mha")
};

struct M2Unit {
  int kv0, kvlen, q0, qrows, sa, sb, h;  // qrows == 0: no unit (queue ran dry)
};

constexpr uint32_t M2_NONE = 0xFFFFFFu;

__device__ __forceinline__ M2Unit m2_unit(const Mha2Params& p, uint32_t u) {
  if (u == M2_NONE) return M2Unit{0, 0, 0, 0, -1, -1, 0};
  const int it = static_cast<int>(u) / p.heads;
  const int4 e = __ldg(p.items + 2 * it);
  const int4 f = __ldg(p.items + 2 * it + 1);
  return M2Unit{e.x, e.y - e.x, e.z, e.w - e.z, f.x, f.y, static_cast<int>(u) - it * p.heads};
}

__device__ __forceinline__ void m2_tie(uint32_t (&r)[32]) {
  asm volatile(""
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                 "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]),
                 "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]),
                 "+r"(r[29]), "+r"(r[30]), "+r"(r[31]));
}

__global__ void __launch_bounds__(M2_THREADS, 2) mha2_fwd_kernel(const __grid_constant__ CUtensorMap tm,
                                                                 const Mha2Params p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sQ = smem + M2Smem::Q_OFF;
  uint8_t* sKV = smem + M2Smem::KV_OFF;
  uint8_t* sOut = smem + M2Smem::OUT_OFF;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + M2Smem::BAR_OFF);
  uint64_t* q_full = bars;        // [2] Q of unit t landed in buffer t & 1
  uint64_t* q_empty = bars + 2;   // [2] the last S MMA of the buffer's unit has read it
  uint64_t* kv_full = bars + 4;   // [2] K block landed in ring slot
  uint64_t* v_full = bars + 6;    // [2] V block landed
  uint64_t* kv_empty = bars + 8;  // [2] P V of the slot's block done: slot free
  uint64_t* s_full = bars + 10;   // S(g) in TMEM
  uint64_t* s_read = bars + 11;   // the softmax holds S(g) in registers: S columns free
  uint64_t* p_full = bars + 12;   // P(g) in TMEM (and O rescaled): issue P(g) V(g)
  uint64_t* pv_done = bars + 13;  // P(g) V(g) accumulated into O: P columns free
  uint64_t* o_free = bars + 14;   // the softmax has read O of its unit: the next unit's first P V may overwrite it
  uint32_t* holder = reinterpret_cast<uint32_t*>(bars + 15);
  uint32_t* ring = holder + 1;  // [4] claimed units, (t & 0xFF) << 24 | unit, polled with smem atomics

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    ptx::prefetch_tmap(&tm);
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&q_full[i], 1);
      ptx::mbar_init(&q_empty[i], 1);
      ptx::mbar_init(&kv_full[i], 1);
      ptx::mbar_init(&v_full[i], 1);
      ptx::mbar_init(&kv_empty[i], 1);
    }
    ptx::mbar_init(s_full, 1);
    ptx::mbar_init(s_read, 128);
    ptx::mbar_init(p_full, 128);
    ptx::mbar_init(pv_done, 1);
    ptx::mbar_init(o_free, 128);
    for (int i = 0; i < 4; ++i) ring[i] = 0xFFFFFFFFu;  // tag 0xFF: nothing published yet
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
  constexpr uint32_t S_COL = 0, P_COL = 128, O_COL = 192;
  ptx::griddep_launch_dependents();
  // qkv, the item list and the claim queue come from earlier kernels of the
  // stream (PDL orders only the immediate predecessor): read after the wait
  ptx::griddep_wait();
  const int nunits = __ldg(p.header) * p.heads;
  const bool active = static_cast<int>(blockIdx.x) < nunits;

  // the t-th unit of this CTA as published by the producer warp
  auto unit_at = [&](int t) -> M2Unit {
    uint32_t v;
    while (((v = atomicAdd(ring + (t & 3), 0u)) >> 24) != (static_cast<uint32_t>(t) & 0xFFu)) {
    }
    return m2_unit(p, v & 0xFFFFFFu);
  };

  if (!active) {
    // no unit for this CTA: straight to the teardown
  } else if (warp >= 4) {
    ptx::setmaxnreg_dec<M2_REGS_ISSUE>();
    if (warp == 4) {
      // ------------------------------------------------ TMA producer
      int kvg = 0;  // K / V blocks loaded so far (ring position)
      for (int t = 0;; ++t) {
        uint32_t u = blockIdx.x;
        if (t > 0) {
          // claim the next unit once this CTA's loads for the current one are
          // all issued: the CTA still has ~1-2 blocks of softmax and an
          // epilogue to go, enough to hide the next unit's Q load and first S
          if (lane == 0) u = gridDim.x + atomicAdd(p.queue, 1);
          u = __shfl_sync(0xffffffffu, u, 0);
          if (u >= static_cast<uint32_t>(nunits)) u = M2_NONE;
        }
        if (lane == 0) atomicExch(ring + (t & 3), (static_cast<uint32_t>(t) & 0xFFu) << 24 | u);
        __syncwarp();
        if (u == M2_NONE) break;
        const M2Unit w = m2_unit(p, u);
        const int qb = t & 1;
        if (t >= 2) ptx::mbar_wait(&q_empty[qb], ((t - 2) >> 1) & 1);  // unit t-2's S MMAs are done with this buffer
        if (ptx::elect_one()) {
          ptx::mbar_arrive_expect_tx(&q_full[qb], M2_TILE);
          ptx::tma_load_2d(sQ + qb * M2_TILE, &tm, &q_full[qb], w.h * M2_D, w.q0);
        }
        __syncwarp();
        const int nkb = (w.kvlen + M2_BLK - 1) / M2_BLK;
        for (int j = 0; j < nkb; ++j, ++kvg) {
          const int slot = kvg & 1;
          ptx::mbar_wait(&kv_empty[slot], ((kvg >> 1) & 1) ^ 1u);
          if (ptx::elect_one()) {
            uint8_t* dst = sKV + slot * 2 * M2_TILE;
            ptx::mbar_arrive_expect_tx(&kv_full[slot], M2_TILE);
            ptx::tma_load_2d(dst, &tm, &kv_full[slot], p.hidden + w.h * M2_D, w.kv0 + j * M2_BLK);
            ptx::mbar_arrive_expect_tx(&v_full[slot], M2_TILE);
            ptx::tma_load_2d(dst + M2_TILE, &tm, &v_full[slot], 2 * p.hidden + w.h * M2_D, w.kv0 + j * M2_BLK);
          }
          __syncwarp();
        }
      }
    } else if (warp == 5) {
      // ------------------------------------------------ MMA issuer
      constexpr uint32_t idesc_s = ptx::idesc_bf16(128, M2_BLK, false, false);  // Q K^T, both K-major
      constexpr uint32_t idesc_o = ptx::idesc_bf16(128, M2_D, false, true);     // P (TMEM) x V (MN-major)
      const uint32_t q_base = ptx::smem_u32(sQ), kv_base = ptx::smem_u32(sKV);
      struct Blk {
        int g, slot, j, t, valid;
        uint32_t par;
      };
      auto issue_pv = [&](const Blk& b) {
        ptx::mbar_wait(&v_full[b.slot], b.par);
        ptx::mbar_wait(p_full, b.g & 1);
        if (b.j == 0 && b.t > 0) ptx::mbar_wait(o_free, (b.t - 1) & 1);  // the previous unit's O has been read
        ptx::tc_fence_after();
        const int nks = (b.valid + 15) / 16;  // only the 16-key steps that hold keys
        const uint64_t v_desc = ptx::sdesc_sw128(kv_base + b.slot * 2 * M2_TILE + M2_TILE, 1024, M2_TILE);
        if (ptx::elect_one()) {
          for (int ks = 0; ks < nks; ++ks)
            ptx::mma_bf16_ts(tmem + O_COL, tmem + P_COL + 8 * ks, v_desc + ks * ((16 * 128) >> 4), idesc_o,
                             (b.j > 0 || ks > 0) ? 1u : 0u);
          ptx::mma_commit(pv_done);
          ptx::mma_commit(&kv_empty[b.slot]);
        }
        __syncwarp();
      };
      int g = 0;
      Blk prev{0, 0, 0, 0, 0, 0u};
      for (int t = 0;; ++t) {
        const M2Unit w = unit_at(t);
        if (w.qrows == 0) break;
        const int qb = t & 1;
        const int nkb = (w.kvlen + M2_BLK - 1) / M2_BLK;
        ptx::mbar_wait(&q_full[qb], (t >> 1) & 1);
        const uint64_t q_desc = ptx::sdesc_sw128(q_base + qb * M2_TILE, 1024, 16);
        for (int j = 0; j < nkb; ++j, ++g) {
          const int slot = g & 1;
          const uint32_t par = static_cast<uint32_t>((g >> 1) & 1);
          ptx::mbar_wait(&kv_full[slot], par);
          if (g > 0) ptx::mbar_wait(s_read, (g - 1) & 1);  // S(g-1) is in the softmax registers
          ptx::tc_fence_after();
          const uint64_t k_desc = ptx::sdesc_sw128(kv_base + slot * 2 * M2_TILE, 1024, 16);
          if (ptx::elect_one()) {
#pragma unroll
            for (int kk = 0; kk < M2_D / 16; ++kk)
              ptx::mma_bf16_ss(tmem + S_COL, q_desc + 2 * kk, k_desc + 2 * kk, idesc_s, kk > 0);
            ptx::mma_commit(s_full);
            if (j == nkb - 1) ptx::mma_commit(&q_empty[qb]);
          }
          __syncwarp();
          if (g > 0) issue_pv(prev);
          prev = Blk{g, slot, j, t, min(M2_BLK, w.kvlen - j * M2_BLK), par};
        }
      }
      if (g > 0) issue_pv(prev);
    }
  } else {
    ptx::setmaxnreg_inc<M2_REGS_SOFTMAX>();
    // ------------------------------------------------ softmax + epilogue
    const int row = threadIdx.x;  // query row of the tile == TMEM lane
    const uint32_t trow = tmem + (static_cast<uint32_t>(warp * 32) << 16);
    const float sl2 = p.sl2;
    int g = 0;
    for (int t = 0;; ++t) {
      const M2Unit w = unit_at(t);
      if (w.qrows == 0) break;
      const int nkb = (w.kvlen + M2_BLK - 1) / M2_BLK;
      const bool warp_live = warp * 32 < w.qrows;
      const bool row_ok = row < w.qrows;
      // my keys [ks, ke) relative to the unit's first key: a group's rows
      // see only their own sequence
      int ks = 0, ke = w.kvlen;
      const bool grouped = w.sa < w.sb;
      if (grouped) {
        if (row_ok) {
          const int r = w.q0 + row;
          int lo = w.sa, hi = w.sb;
          while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (__ldg(p.seq_starts + mid) <= r) lo = mid; else hi = mid - 1;
          }
          ks = __ldg(p.seq_starts + lo) - w.kv0;
          ke = __ldg(p.seq_starts + lo + 1) - w.kv0;
        } else {
          ks = ke = 0;
        }
      }
      float mref = -INFINITY, lsum = 0.f;
      for (int j = 0; j < nkb; ++j, ++g) {
        const int klo = ks - j * M2_BLK, khi = min(ke - j * M2_BLK, M2_BLK);  // my valid keys of this block
        ptx::mbar_wait(s_full, g & 1);
        ptx::tc_fence_after();
        // Pass 1: the row max, 64 scores at a time (a thread holds a whole
        // row: 128 scores would not fit next to the pipeline's registers at
        // two CTAs per SM).  Pass 2 reloads each half for its exponentials;
        // TMEM reads are cheap (~860 B/clk/SM measured, scripts/micro/tmem_bw.cu).
        const bool masked = klo > 0 || khi < M2_BLK;
        auto mask64 = [&](uint32_t (&a)[32], uint32_t (&b)[32], int base) {
          // keys outside my row's problem: s = -inf (out of the max; exp -> 0)
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            if (base + i < klo || base + i >= khi) a[i] = 0xff800000u;
            if (base + 32 + i < klo || base + 32 + i >= khi) b[i] = 0xff800000u;
          }
        };
        bool need = false;
        float alpha = 1.f;
        if (warp_live) {
          float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
          for (int hf = 0; hf < 2; ++hf) {
            uint32_t a[32], b[32];
            ptx::tmem_ld32(trow + S_COL + 64 * hf, a);
            ptx::tmem_ld32(trow + S_COL + 64 * hf + 32, b);
            ptx::tmem_wait_ld(a);
            m2_tie(b);
            if (masked) mask64(a, b, 64 * hf);
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              m4[0] = ptx::max3(m4[0], __uint_as_float(a[i]), __uint_as_float(a[i + 1]));
              m4[1] = ptx::max3(m4[1], __uint_as_float(a[i + 2]), __uint_as_float(a[i + 3]));
              m4[2] = ptx::max3(m4[2], __uint_as_float(b[i]), __uint_as_float(b[i + 1]));
              m4[3] = ptx::max3(m4[3], __uint_as_float(b[i + 2]), __uint_as_float(b[i + 3]));
            }
          }
          const float bmax = fmaxf(ptx::max3(m4[0], m4[1], m4[2]), m4[3]);
          const float mnew = fmaxf(mref, bmax);
          need = (mnew - mref) * sl2 > M2_RESCALE_LOG2;  // true on the first block with a key (mref = -inf)
          alpha = (need && mref != -INFINITY) ? ptx::ex2_approx((mref - mnew) * sl2) : 1.f;
          if (need) mref = mnew;
        }
        if (j > 0) {
          ptx::mbar_wait(pv_done, (g - 1) & 1);  // P(g-1) V(g-1) is in O; the P columns are free
          ptx::tc_fence_after();
        }
        if (warp_live && __any_sync(0xffffffffu, need && j > 0)) {
          // the reference max moved (rare): my O row *= 2^((m_old - m_new) * scale)
          const unsigned long long a2 = ptx::f2(alpha, alpha);
#pragma unroll
          for (int hf = 0; hf < 2; ++hf) {
            uint32_t o[32];
            ptx::tmem_ld32(trow + O_COL + 32 * hf, o);
            ptx::tmem_wait_ld(o);
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
              float a, c;
              ptx::unf2(ptx::mul2(ptx::f2(__uint_as_float(o[i]), __uint_as_float(o[i + 1])), a2), a, c);
              o[i] = __float_as_uint(a);
              o[i + 1] = __float_as_uint(c);
            }
            ptx::tmem_st32(trow + O_COL + 32 * hf, o);
          }
        }
        // Pass 2: P = 2^((s - m_ref) * scale * log2 e), 64 keys at a time.
        // (a row with no key in the blocks so far keeps m_ref = -inf; its
        // scores are all -inf, so any finite offset gives P = 0)
        const float msc = (mref == -INFINITY) ? 0.f : mref * sl2;
        const unsigned long long sl2x2 = ptx::f2(sl2, sl2), nm2 = ptx::f2(-msc, -msc);
        unsigned long long sum4[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          uint32_t a[32], b[32];
          if (warp_live) {
            ptx::tmem_ld32(trow + S_COL + 64 * hf, a);
            ptx::tmem_ld32(trow + S_COL + 64 * hf + 32, b);
            ptx::tmem_wait_ld(a);
            m2_tie(b);
          }
          if (hf == 1) {
            ptx::tc_fence_before();
            ptx::mbar_arrive(s_read);  // every S value is read: the MMA warp may write the next block's S
          }
          if (!warp_live) continue;
          if (masked) mask64(a, b, 64 * hf);
#pragma unroll
          for (int c2 = 0; c2 < 2; ++c2) {
            uint32_t (&v)[32] = c2 == 0 ? a : b;
            const int key0 = 64 * hf + 32 * c2;
            uint32_t pp[16];  // 32 keys as bf16 pairs -> P columns key0 / 2 ..
            const bool empty = key0 >= khi || key0 + 32 <= klo;
            if (__all_sync(0xffffffffu, empty)) {  // no key of any row here: P = 0, no exponentials
#pragma unroll
              for (int i = 0; i < 16; ++i) pp[i] = 0u;
            } else {
#pragma unroll
              for (int i = 0; i < 32; i += 2) {
                float x0, x1, e0, e1;
                ptx::unf2(ptx::fma2(ptx::f2(__uint_as_float(v[i]), __uint_as_float(v[i + 1])), sl2x2, nm2), x0, x1);
                if ((i & 15) < BT_MHA2_POLY) {
                  ptx::ex2_poly2(x0, x1, e0, e1);  // masked key (x = -inf): exactly 0
                } else {
                  e0 = ptx::ex2_approx(x0);  // ex2(-inf) = 0
                  e1 = ptx::ex2_approx(x1);
                }
                sum4[(i >> 1) & 3] = ptx::add2(sum4[(i >> 1) & 3], ptx::f2(e0, e1));
                pp[i / 2] = ptx::pack_bf16x2(e0, e1);
              }
            }
            ptx::tmem_st16(trow + P_COL + key0 / 2, pp);
          }
        }
        if (warp_live) {
          const unsigned long long bsum2 = ptx::add2(ptx::add2(sum4[0], sum4[1]), ptx::add2(sum4[2], sum4[3]));
          float s0f, s1f;
          ptx::unf2(bsum2, s0f, s1f);
          lsum = lsum * alpha + (s0f + s1f);
          ptx::tmem_wait_st();
        }
        ptx::tc_fence_before();
        ptx::mbar_arrive(p_full);
      }
      // ---- epilogue: O / l -> bf16 rows -> staging -> 16-byte coalesced stores
      ptx::mbar_wait(pv_done, (g - 1) & 1);  // this unit's last P V
      ptx::tc_fence_after();
      uint32_t o0[32], o1[32];
      if (warp_live) {
        ptx::tmem_ld32(trow + O_COL, o0);
        ptx::tmem_ld32(trow + O_COL + 32, o1);
        ptx::tmem_wait_ld(o0);
        m2_tie(o1);
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(o_free);  // the next unit's first P V may overwrite O
      if (warp_live) {
        const float inv = row_ok ? 1.0f / lsum : 0.f;
        const unsigned long long inv2 = ptx::f2(inv, inv);
        uint8_t* mine = sOut + row * 128;
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          uint32_t wv[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int k = 8 * jj + 2 * e;
            const uint32_t lo = k < 32 ? o0[k] : o1[k - 32], hi = k < 32 ? o0[k + 1] : o1[k - 31];
            float a, b2;
            ptx::unf2(ptx::mul2(ptx::f2(__uint_as_float(lo), __uint_as_float(hi)), inv2), a, b2);
            wv[e] = ptx::pack_bf16x2(a, b2);
          }
          *reinterpret_cast<uint4*>(mine + ((jj ^ (row & 7)) << 4)) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
        }
        __syncwarp();  // this warp's 32 rows are staged
        // lane -> (row of the warp's slab, 16 B chunk): 4 rows per store instruction
#pragma unroll
        for (int it = 0; it < 8; ++it) {
          const int rr = warp * 32 + it * 4 + (lane >> 3);
          const int jj = lane & 7;
          if (rr < w.qrows) {
            const uint4 v = *reinterpret_cast<const uint4*>(sOut + rr * 128 + ((jj ^ (rr & 7)) << 4));
            *reinterpret_cast<uint4*>(p.out + static_cast<size_t>(w.q0 + rr) * p.hidden + w.h * M2_D + jj * 8) = v;
          }
        }
        __syncwarp();  // the slab is read: the next unit may stage into it
        if (p.flops != nullptr) {
          // instrumentation: 4 * d FLOPs per (row, key of its own problem)
          const unsigned keys = row_ok ? static_cast<unsigned>(ke - ks) : 0u;
          const unsigned sumk = __reduce_add_sync(0xffffffffu, keys);
          if (lane == 0 && sumk) atomicAdd(p.flops, 4ull * M2_D * sumk);
        }
      }
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 256);
  }
  if (active && threadIdx.x == 0) {
    // every claim of this CTA precedes this point; the last CTA to finish
    // resets the queue for the next launch (the next forward's plan also
    // zeroes it)
    const int participants = min(static_cast<int>(gridDim.x), nunits);
    __threadfence();
    if (atomicAdd(p.queue + 1, 1) == participants - 1) {
      p.queue[0] = 0;
      p.queue[1] = 0;
      __threadfence();
    }
  }
}

extern unsigned long long* g_mha_flops;

// Resident CTAs per SM: from shared memory, registers and TMEM (the occupancy
// API under-reports these warp-specialised kernels, see mha_sm100.cu).
static int mha2_slots() {
  static int slots = 0;
  if (slots == 0) {
    BT_CUDA_CHECK(cudaFuncSetAttribute(mha2_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(M2Smem::SMEM)));
    BT_CUDA_CHECK(cudaFuncSetAttribute(mha2_fwd_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    int dev = 0, sm_smem = 0, rsv = 0;
    BT_CUDA_CHECK(cudaGetDevice(&dev));
    BT_CUDA_CHECK(cudaDeviceGetAttribute(&sm_smem, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev));
    BT_CUDA_CHECK(cudaDeviceGetAttribute(&rsv, cudaDevAttrReservedSharedMemoryPerBlock, dev));
    const int by_smem = sm_smem / static_cast<int>(M2Smem::SMEM + rsv);
    const int per_sm = std::min(by_smem, 2);  // TMEM: 256 columns each
    BT_REQUIRE(per_sm >= 1, BT_ECUDA, "mha2: the kernel does not fit on an SM");
    slots = per_sm * (num_sms() > 0 ? num_sms() : 148);
  }
  return slots;
}

static int g_mha2_grid = 0;  // test hook: pin the persistent grid (0 = the resident slots)

// The forward's MHA: the persistent kernel over bt_plan_sched's items.
int mha2_launch(const void* qkv, const int32_t* seq_starts, const void* sched, int bs, int mx, int H, int d, int T,
                void* out, cudaStream_t s) {
  BT_REQUIRE(d == M2_D, BT_ECONFIG, "fused MHA supports head_size 64, got %d", d);
  BT_REQUIRE(bs >= 1 && mx >= 1 && H >= 1 && T >= 1 && sched, BT_ESHAPE, "mha2: bad arguments");
  const int hidden = H * d;
  CUtensorMap tm;
  BT_TRY(make_tmap_bf16_2d(&tm, qkv, T, 3 * hidden, 3 * hidden, 128, 64));
  Mha2Params p;
  p.out = static_cast<__nv_bfloat16*>(out);
  p.seq_starts = seq_starts;
  p.header = reinterpret_cast<const int*>(static_cast<const uint8_t*>(sched) + sched_segs_offset(bs, mx));
  p.items = reinterpret_cast<const int4*>(p.header + 4);
  p.queue = const_cast<int*>(p.header + 1);
  p.hidden = hidden;
  p.heads = H;
  p.sl2 = 1.4426950408889634f / sqrtf(static_cast<float>(d));
  p.flops = g_mha_flops;
  const int slots = mha2_slots();
  const long long max_units = static_cast<long long>(bs) * ((mx + 127) / 128) * H;
  int grid = g_mha2_grid > 0 ? g_mha2_grid : slots;
  if (max_units < grid) grid = static_cast<int>(max_units);
  BT_LAUNCH(mha2_fwd_kernel, dim3(grid), dim3(M2_THREADS), M2Smem::SMEM, s, 1, tm, p);
  return BT_OK;
}

}  // namespace bt

// Test hook: pin the persistent MHA grid (0 = one CTA per resident slot).
extern "C" int bt_debug_mha2_grid(int grid) {
  BT_REQUIRE(grid >= 0, BT_ECONFIG, "bt_debug_mha2_grid: grid >= 0");
  bt::g_mha2_grid = grid;
  return BT_OK;
}
