// Fused variable-length MHA, four-CTAs-per-SM kernel (what the forward runs
// outside the small-batch segment kernel; BT_MHA64=0 restores the two-CTA
// kernels of mha_sm100.cu): the same math as mha_fwd_kernel (reference attention.py:177-314,
// single-pass softmax with a lazily moved reference max, P never leaving the
// SM) restructured so that FOUR query tiles run per SM instead of two.
//
//   * 64-key blocks: TMEM per CTA = S [0,64) fp32 + O [64,128) fp32 = 128
//     columns; P (bf16 pairs) is written over S columns [0,32) once the
//     softmax holds S in registers, so four CTAs fit the 512 columns.
//   * thread = query row (warps 0-3, TMEM lane = thread): row max and row
//     sum are thread-local, no shuffles, 64 S values per thread.
//   * the MMA warp issues S(j+1) right behind P(j) V(j) (they share
//     columns; MMAs of one thread execute in order); the four CTAs keep the SFU busy
//     while a CTA waits for its MMAs -- the two-CTA kernel's chain is gated
//     by two all-thread barriers per 128-key block with only two chains per SM.
//   * O is rescaled (rarely) after block j's exponentials, before P(j) is
//     released: S(j)'s commit also covered P(j-1) V(j-1) (a commit tracks
//     every prior tcgen05 op of the issuing thread), so O is stable then.
//
// One CTA per (128-row query tile, head, sequence), longest sequences first
// (bt_plan_sched); tiles past a sequence's end exit at once.  d = 64.

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "ptx.cuh"
#include "tma_host.cuh"

namespace bt {

constexpr int M64_D = 64;
constexpr int M64_QT = 128;
constexpr int M64_KB = 64;
constexpr uint32_t M64_QTILE = 128 * 128;  // 128 rows x 64 bf16
constexpr uint32_t M64_KVTILE = 64 * 128;  // 64 rows x 64 bf16
#ifndef BT_M64_NST
#define BT_M64_NST 2  // K/V ring depth (2: four CTAs fit an SM's shared memory)
#endif
#ifndef BT_M64_CTAS
#define BT_M64_CTAS 4  // resident CTAs per SM the launch bounds target
#endif
constexpr int M64_NST = BT_M64_NST;
constexpr int M64_THREADS = 256;
// register split (setmaxnreg): the single-tile kernel's issue warps fit in
// 24, giving the softmax warpgroup 104 (128 x 104 + 128 x 24 = 256 x 64); the
// persistent kernel's issue loops need 32 (softmax 96)
template <bool PERSIST>
struct M64Regs {
  static constexpr int ISSUE = PERSIST ? 32 : 24;
  static constexpr int SOFTMAX = PERSIST ? 96 : 104;
};
constexpr uint32_t M64_KV_OFF = M64_QTILE;
constexpr uint32_t M64_BAR_OFF = M64_KV_OFF + M64_NST * 2 * M64_KVTILE;
constexpr size_t M64_SMEM = M64_BAR_OFF + 256;

#ifndef BT_MHA_POLY
#define BT_MHA_POLY 2
#endif

struct Mha64Params {
  const int32_t* seq_starts;
  // optional (the forward's schedule, bt_plan_sched): *nunits query-tile
  // units {start row, qt << 20 | length}, longest sequences first; item i =
  // (unit i / heads, head i % heads).  With it the grid is persistent: CTA c
  // works items c, c + G, c + 2G, ...  Without it: one tile per CTA, grid
  // (query tile, head, sequence) over seq_starts.
  const int2* units;
  const int* nunits;
  // optional (grid mode): CTA z -> (start row, length), longest first
  const int2* order;
  int heads;
  __nv_bfloat16* out;
  int hidden;
  float sl2;
  unsigned long long* flops;
};

// Debug trace (a -DBT_TRACE_ON build, buffer installed by bt_debug_mha_trace;
// grid mode, the CTA's tile): 32 u64 globaltimer stamps per CTA, index =
// linear block id.  [0] set-up done  [1] Q landed (MMA warp)  block j < 7:
// [2+2j] S(j) seen by the softmax  [3+2j] P(j) released  [16+j] P(j) seen by
// the MMA warp (P V(j) issued)  [30] O seen  [31] output stored.
__device__ unsigned long long* g_m64_trace = nullptr;
#ifdef BT_TRACE_ON
#define M64_TRACE(slot)                                                                                  \
  do {                                                                                                   \
    if (g_m64_trace) {                                                                                   \
      unsigned long long _t;                                                                             \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));                                             \
      g_m64_trace[((blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) * 32 + (slot)] = _t;  \
    }                                                                                                    \
  } while (0)
#else
#define M64_TRACE(slot) \
  do {                  \
  } while (0)
#endif
int mha64_set_trace(unsigned long long* buf) {
  BT_CUDA_CHECK(cudaMemcpyToSymbol(g_m64_trace, &buf, sizeof(buf)));
  return BT_OK;
}

struct M64Tile {
  int s0, len, q0, h;  // keys [s0, s0 + len); query rows s0 + q0 .. ; len 0: no tile
};

__device__ __forceinline__ void m64_tie(uint32_t (&r)[32]) {
  asm volatile(""
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                 "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]),
                 "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]),
                 "+r"(r[29]), "+r"(r[30]), "+r"(r[31]));
}

// PERSIST = true: a persistent grid walking the plan's query-tile units
// (launches of many waves); false: one tile per CTA, grid (tile, head,
// sequence) -- the single-tile code path without the loop's bookkeeping.
template <bool PERSIST>
__global__ void __launch_bounds__(M64_THREADS, BT_M64_CTAS)
    mha64_fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmKV,
                     const Mha64Params p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sQ = smem;
  uint8_t* sKV = smem + M64_KV_OFF;  // slot s: K at +16K*s, V at +16K*s + 8K
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + M64_BAR_OFF);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;
  uint64_t* v_full = k_full + M64_NST;
  uint64_t* k_empty = v_full + M64_NST;
  uint64_t* v_empty = k_empty + M64_NST;
  uint64_t* s_full = v_empty + M64_NST;  // S(j) in TMEM (and every earlier MMA done)
  uint64_t* p_full = s_full + 1;         // P(j) written over S by all 128 softmax threads
  uint64_t* o_full = s_full + 2;         // a tile's last P V done
  uint64_t* o_free = s_full + 3;         // the softmax has read a tile's O (the next tile may overwrite it)
  uint64_t* q_free = s_full + 4;         // a tile's last S MMA done with Q (the next Q may land)
  uint32_t* holder = reinterpret_cast<uint32_t*>(q_free + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    ptx::prefetch_tmap(&tmQ);
    ptx::prefetch_tmap(&tmKV);
    ptx::mbar_init(q_full, 1);
    for (int i = 0; i < M64_NST; ++i) {
      ptx::mbar_init(&k_full[i], 1);
      ptx::mbar_init(&v_full[i], 1);
      ptx::mbar_init(&k_empty[i], 1);
      ptx::mbar_init(&v_empty[i], 1);
    }
    ptx::mbar_init(s_full, 1);
    ptx::mbar_init(p_full, 128);
    ptx::mbar_init(o_full, 1);
    ptx::mbar_init(o_free, 128);
    ptx::mbar_init(q_free, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 0) {
    ptx::tmem_alloc(holder, 128);
    ptx::tmem_relinquish();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *holder;
  ptx::griddep_launch_dependents();
  ptx::griddep_wait();  // the schedule and qkv come from earlier kernels
  if (!PERSIST && threadIdx.x == 0) M64_TRACE(0);
  constexpr bool persistent = PERSIST;
  const int nitems = persistent ? __ldg(p.nunits) * p.heads : 1;
  constexpr int max_tiles = PERSIST ? 0x7FFFFFFF : 1;
  // the t-th tile of this CTA (len 0: none)
  auto tile_at = [&](int t) -> M64Tile {
    if (persistent) {
      const int item = static_cast<int>(blockIdx.x) + t * static_cast<int>(gridDim.x);
      if (item >= nitems) return M64Tile{0, 0, 0, 0};
      const int u = item / p.heads;
      const int2 e = __ldg(p.units + u);
      return M64Tile{e.x, e.y & 0xFFFFF, (e.y >> 20) * M64_QT, item - u * p.heads};
    }
    if (t > 0) return M64Tile{0, 0, 0, 0};
    const int b = blockIdx.z;
    int sb, len;
    if (p.order != nullptr) {
      const int2 e = __ldg(p.order + b);
      sb = e.x;
      len = e.y;
    } else {
      sb = __ldg(p.seq_starts + b);
      len = __ldg(p.seq_starts + b + 1) - sb;
    }
    const int q0 = blockIdx.x * M64_QT;
    return q0 < len ? M64Tile{sb, len, q0, static_cast<int>(blockIdx.y)} : M64Tile{0, 0, 0, 0};
  };
  constexpr uint32_t S_COL = 0, O_COL = 64;

  if (tile_at(0).len == 0) {
    // CTA-uniform: no work
  } else if (warp >= 4) {
    ptx::setmaxnreg_dec<M64Regs<PERSIST>::ISSUE>();
    if (warp == 4) {
      // ---------------------------------------------- TMA producer
      int kvg = 0;  // K / V blocks loaded so far (ring position across tiles)
      for (int t = 0; t < max_tiles; ++t) {
        const M64Tile tl = tile_at(t);
        if (tl.len == 0) break;
        if (t > 0) ptx::mbar_wait(q_free, static_cast<uint32_t>((t - 1) & 1));  // the last S of tile t-1 read Q
        if (ptx::elect_one()) {
          ptx::mbar_arrive_expect_tx(q_full, M64_QTILE);
          ptx::tma_load_2d(sQ, &tmQ, q_full, tl.h * M64_D, tl.s0 + tl.q0);
        }
        __syncwarp();
        const int nkb = (tl.len + M64_KB - 1) / M64_KB;
        for (int j = 0; j < nkb; ++j, ++kvg) {
          const int slot = kvg % M64_NST;
          const uint32_t ph = static_cast<uint32_t>((kvg / M64_NST) & 1) ^ 1u;
          ptx::mbar_wait(&k_empty[slot], ph);
          if (ptx::elect_one()) {
            ptx::mbar_arrive_expect_tx(&k_full[slot], M64_KVTILE);
            ptx::tma_load_2d(sKV + slot * 2 * M64_KVTILE, &tmKV, &k_full[slot], p.hidden + tl.h * M64_D,
                             tl.s0 + j * M64_KB);
          }
          __syncwarp();
          ptx::mbar_wait(&v_empty[slot], ph);
          if (ptx::elect_one()) {
            ptx::mbar_arrive_expect_tx(&v_full[slot], M64_KVTILE);
            ptx::tma_load_2d(sKV + slot * 2 * M64_KVTILE + M64_KVTILE, &tmKV, &v_full[slot],
                             2 * p.hidden + tl.h * M64_D, tl.s0 + j * M64_KB);
          }
          __syncwarp();
        }
      }
    } else if (warp == 5) {
      // ---------------------------------------------- MMA issuer
      constexpr uint32_t idesc_s = ptx::idesc_bf16(128, M64_KB, false, false);  // Q K^T, both K-major
      constexpr uint32_t idesc_o = ptx::idesc_bf16(128, M64_D, false, true);    // P (TMEM) x V (MN-major)
      const uint64_t q_desc = ptx::sdesc_sw128(ptx::smem_u32(sQ), 1024, 16);
      const uint32_t kv_base = ptx::smem_u32(sKV);
      int kvg = 0, g = 0;  // ring position, blocks issued (S) across tiles
      // S(block j of the current tile) into the S columns -- right behind the
      // previous P V, which read P from them (tcgen05.mma ops of one thread
      // execute in issue order; CUTLASS's Blackwell FMHA aliases P into S
      // the same way); the tile's last S releases Q
      auto issue_s = [&](bool last) {
        const int slot = kvg % M64_NST;
        ptx::mbar_wait(&k_full[slot], static_cast<uint32_t>((kvg / M64_NST) & 1));
        ptx::tc_fence_after();
        const uint64_t k_desc = ptx::sdesc_sw128(kv_base + slot * 2 * M64_KVTILE, 1024, 16);
        if (ptx::elect_one()) {
#pragma unroll
          for (int kk = 0; kk < M64_D / 16; ++kk)
            ptx::mma_bf16_ss(tmem + S_COL, q_desc + 2 * kk, k_desc + 2 * kk, idesc_s, kk > 0);
          ptx::mma_commit(&k_empty[slot]);
          ptx::mma_commit(s_full);
          if (PERSIST && last) ptx::mma_commit(q_free);
        }
        __syncwarp();
      };
      for (int t = 0; t < max_tiles; ++t) {
        const M64Tile tl = tile_at(t);
        if (tl.len == 0) break;
        const int nkb = (tl.len + M64_KB - 1) / M64_KB;
        ptx::mbar_wait(q_full, static_cast<uint32_t>(t & 1));
        if (!PERSIST && lane == 0) M64_TRACE(1);
        const int kv0 = kvg;
        issue_s(nkb == 1);
        for (int j = 0; j < nkb; ++j, ++g) {
          const int slot = (kv0 + j) % M64_NST;
          ptx::mbar_wait(p_full, static_cast<uint32_t>(g & 1));
          if (!PERSIST && lane == 0 && j < 7) M64_TRACE(16 + j);
          if (PERSIST && j == 0 && t > 0)
            ptx::mbar_wait(o_free, static_cast<uint32_t>((t - 1) & 1));  // O of tile t-1 read
          ptx::mbar_wait(&v_full[slot], static_cast<uint32_t>(((kv0 + j) / M64_NST) & 1));
          ptx::tc_fence_after();
          const int keys = min(M64_KB, tl.len - j * M64_KB);
          const int nks = (keys + 15) / 16;
          const uint64_t v_desc =
              ptx::sdesc_sw128(kv_base + slot * 2 * M64_KVTILE + M64_KVTILE, 1024, M64_KVTILE);
          if (ptx::elect_one()) {
            for (int ks = 0; ks < nks; ++ks)
              ptx::mma_bf16_ts(tmem + O_COL, tmem + S_COL + 8 * ks, v_desc + ks * ((16 * 128) >> 4), idesc_o,
                               (j > 0 || ks > 0) ? 1u : 0u);
            ptx::mma_commit(&v_empty[slot]);
            if (j + 1 == nkb) ptx::mma_commit(o_full);
          }
          __syncwarp();
          if (j + 1 < nkb) {
            ++kvg;
            issue_s(j + 2 == nkb);
          }
        }
        ++kvg;  // the tile's last block
      }
    }
  } else {
    ptx::setmaxnreg_inc<M64Regs<PERSIST>::SOFTMAX>();
    // ------------------------------------------------ softmax, thread = row
    const int row = threadIdx.x;  // TMEM lane
    const uint32_t trow = tmem + (static_cast<uint32_t>(warp * 32) << 16);
    const float sl2 = p.sl2;
    int g = 0;  // blocks consumed across tiles
    for (int t = 0; t < max_tiles; ++t) {
      int len, rows_here;
      M64Tile tl0 = tile_at(t);  // (persistent: s0, h re-read at the store -- fewer live registers)
      len = tl0.len;
      rows_here = tl0.len - tl0.q0;
      if (len == 0) break;
      const int nkb = (len + M64_KB - 1) / M64_KB;
      const bool warp_live = warp * 32 < rows_here;
      float mref = -INFINITY, lsum = 0.f;
      for (int j = 0; j < nkb; ++j, ++g) {
        const int kblk = min(M64_KB, len - j * M64_KB);
        ptx::mbar_wait(s_full, static_cast<uint32_t>(g & 1));
        ptx::tc_fence_after();
        if (!PERSIST && threadIdx.x == 0 && j < 7) M64_TRACE(2 + 2 * j);
        uint32_t r0[32], r1[32];
        if (warp_live) {
          ptx::tmem_ld32(trow + S_COL, r0);
          ptx::tmem_ld32(trow + S_COL + 32, r1);
          ptx::tmem_wait_ld(r0);
          m64_tie(r1);
          if (kblk < 64) {  // keys past the sequence end: -inf (exp -> exactly 0)
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              if (i >= kblk) r0[i] = 0xff800000u;
              if (32 + i >= kblk) r1[i] = 0xff800000u;
            }
          }
          float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            m4[0] = ptx::max3(m4[0], __uint_as_float(r0[i]), __uint_as_float(r0[i + 1]));
            m4[1] = ptx::max3(m4[1], __uint_as_float(r0[i + 2]), __uint_as_float(r0[i + 3]));
            m4[2] = ptx::max3(m4[2], __uint_as_float(r1[i]), __uint_as_float(r1[i + 1]));
            m4[3] = ptx::max3(m4[3], __uint_as_float(r1[i + 2]), __uint_as_float(r1[i + 3]));
          }
          const float bmax = fmaxf(ptx::max3(m4[0], m4[1], m4[2]), m4[3]);
          const float mnew = fmaxf(mref, bmax);
          const bool need = (mnew - mref) * sl2 > 8.0f;  // true on the first block
          float alpha = 1.f;
          if (need) {
            alpha = mref != -INFINITY ? ptx::ex2_approx((mref - mnew) * sl2) : 1.f;
            mref = mnew;
            lsum *= alpha;
          }
          const float msc = mref * sl2;
          const unsigned long long sl2x2 = ptx::f2(sl2, sl2), nm2 = ptx::f2(-msc, -msc);
          unsigned long long sum4[4] = {0ull, 0ull, 0ull, 0ull};
          auto exps = [&](const uint32_t (&r)[32], uint32_t (&pp)[16]) {
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
              float x0, x1, e0, e1;
              ptx::unf2(ptx::fma2(ptx::f2(__uint_as_float(r[i]), __uint_as_float(r[i + 1])), sl2x2, nm2), x0, x1);
              if ((i & 15) < BT_MHA_POLY) {
                ptx::ex2_poly2(x0, x1, e0, e1);
              } else {
                e0 = ptx::ex2_approx(x0);
                e1 = ptx::ex2_approx(x1);
              }
              sum4[(i >> 1) & 3] = ptx::add2(sum4[(i >> 1) & 3], ptx::f2(e0, e1));
              pp[i / 2] = ptx::pack_bf16x2(e0, e1);
            }
          };
          {
            uint32_t pp[16];
            exps(r0, pp);
            ptx::tmem_st16(trow + S_COL, pp);  // P for keys 0-31 -> columns 0-15
          }
          if (kblk > 32) {
            uint32_t pp[16];
            exps(r1, pp);
            ptx::tmem_st16(trow + S_COL + 16, pp);  // keys 32-63 -> columns 16-31
          } else {
            ptx::tmem_st16_zero(trow + S_COL + 16);  // no key of the problem among keys 32-63
          }
          const unsigned long long s2 = ptx::add2(ptx::add2(sum4[0], sum4[1]), ptx::add2(sum4[2], sum4[3]));
          float sa, sc;
          ptx::unf2(s2, sa, sc);
          lsum += sa + sc;
          if (__any_sync(0xffffffffu, need && j > 0)) {
            // the reference max moved (rare) for some row of the warp: O *=
            // alpha (1 for the other rows) before P(j) V(j) adds to it --
            // warp-uniform, tcgen05.ld / st are warp-collective.  O is
            // stable: S(j)'s commit covered P(j-1) V(j-1).  Done after the
            // exponentials so S and O are never live together.
            const unsigned long long a2 = ptx::f2(alpha, alpha);
#pragma unroll
            for (int half = 0; half < 2; ++half) {
              uint32_t o[32];
              ptx::tmem_ld32(trow + O_COL + 32 * half, o);
              ptx::tmem_wait_ld(o);
#pragma unroll
              for (int i = 0; i < 32; i += 2) {
                float a, c;
                ptx::unf2(ptx::mul2(ptx::f2(__uint_as_float(o[i]), __uint_as_float(o[i + 1])), a2), a, c);
                o[i] = __float_as_uint(a);
                o[i + 1] = __float_as_uint(c);
              }
              ptx::tmem_st32(trow + O_COL + 32 * half, o);
            }
          }
          ptx::tmem_wait_st();
        }
        ptx::tc_fence_before();
        ptx::mbar_arrive(p_full);
        if (!PERSIST && threadIdx.x == 0 && j < 7) M64_TRACE(3 + 2 * j);
      }
      // ---- the tile's output: O / l -> bf16, each thread stores its row
      ptx::mbar_wait(o_full, static_cast<uint32_t>(t & 1));
      ptx::tc_fence_after();
      if (!PERSIST && threadIdx.x == 0) M64_TRACE(30);
      if (warp_live) {
        uint32_t o0[32], o1[32];
        ptx::tmem_ld32(trow + O_COL, o0);
        ptx::tmem_ld32(trow + O_COL + 32, o1);
        ptx::tmem_wait_ld(o0);
        m64_tie(o1);
        if (row < rows_here) {
          const M64Tile tl = PERSIST ? tile_at(t) : tl0;
          const float inv = 1.0f / lsum;
          const unsigned long long inv2 = ptx::f2(inv, inv);
          uint4* dst =
              reinterpret_cast<uint4*>(p.out + static_cast<size_t>(tl.s0 + tl.q0 + row) * p.hidden + tl.h * M64_D);
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const uint32_t* src = c < 4 ? o0 + 8 * c : o1 + 8 * (c - 4);
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              float a, b2;
              ptx::unf2(ptx::mul2(ptx::f2(__uint_as_float(src[2 * e]), __uint_as_float(src[2 * e + 1])), inv2), a,
                        b2);
              w[e] = ptx::pack_bf16x2(a, b2);
            }
            dst[c] = make_uint4(w[0], w[1], w[2], w[3]);
          }
        }
        if (!PERSIST && threadIdx.x == 0) M64_TRACE(31);
        if (p.flops != nullptr) {
          const unsigned keys = row < rows_here ? static_cast<unsigned>(len) : 0u;
          const unsigned wsum = __reduce_add_sync(0xffffffffu, keys);
          if (lane == 0 && wsum) atomicAdd(p.flops, 4ull * M64_D * wsum);
        }
      }
      if constexpr (PERSIST) {
        ptx::tc_fence_before();
        ptx::mbar_arrive(o_free);  // O has been read: the next tile's first P V may overwrite it
      }
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 128);
  }
}

extern unsigned long long* g_mha_flops;

// Every packed-layout MHA launch outside the segment kernel's domain runs this
// kernel (one query tile per CTA, also for launches of many waves: it beats
// the two-CTA kernel's tile list there).  BT_MHA64=0 falls back to the
// two-CTA kernels; bt_debug_mha64 overrides (tests of those kernels' modes).
static int g_mha64_override = -1;
bool mha64_enabled() {
  if (g_mha64_override >= 0) return g_mha64_override == 1;
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("BT_MHA64");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

int mha64_launch(const void* qkv, const int32_t* seq_starts, const void* sched, int bs, int mx, int H, int T,
                 void* out, cudaStream_t s) {
  const int hidden = H * M64_D;
  CUtensorMap tq, tkv;
  BT_TRY(make_tmap_bf16_2d(&tq, qkv, T, 3 * hidden, 3 * hidden, M64_QT, 64));
  BT_TRY(make_tmap_bf16_2d(&tkv, qkv, T, 3 * hidden, 3 * hidden, M64_KB, 64));
  Mha64Params p;
  p.seq_starts = seq_starts;
  p.units = nullptr;
  p.nunits = nullptr;
  p.order = static_cast<const int2*>(sched);  // longest sequences first (bt_plan_sched), or null
  p.heads = H;
  const int sms = num_sms() > 0 ? num_sms() : 148;
  const int nqt_ = (mx + M64_QT - 1) / M64_QT;
  const long long items_max = static_cast<long long>(bs) * nqt_ * H;
  // Launches of many waves (> 4 waves of the 4-per-SM slots) run a persistent
  // grid over the plan's query-tile units: each CTA's next Q load overlaps
  // its previous tile's last block (C5: 2050 -> 1995 us).  Fewer waves keep
  // one tile per CTA, which the hardware hands out dynamically (a static
  // stride over the units balanced C3 worse: 26.6 vs 20.8 us).
  if (sched != nullptr && items_max > 16LL * sms) {
    p.nunits = reinterpret_cast<const int*>(static_cast<const uint8_t*>(sched) + sched_units_offset(bs));
    p.units = reinterpret_cast<const int2*>(p.nunits + 4);
  }
  p.out = static_cast<__nv_bfloat16*>(out);
  p.hidden = hidden;
  p.sl2 = 1.4426950408889634f / sqrtf(static_cast<float>(M64_D));
  p.flops = g_mha_flops;
  static bool set = false;
  if (!set) {
    for (auto kern : {mha64_fwd_kernel<false>, mha64_fwd_kernel<true>}) {
      BT_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(M64_SMEM)));
      BT_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    }
    set = true;
  }
  const int nqt = (mx + M64_QT - 1) / M64_QT;
  if (p.units != nullptr) {
    // persistent: every resident CTA slot (4 per SM), items strided over them
    const int grid = static_cast<int>(std::min<long long>(items_max, 4LL * sms));
    BT_LAUNCH(mha64_fwd_kernel<true>, dim3(grid), dim3(M64_THREADS), M64_SMEM, s, 1, tq, tkv, p);
    return BT_OK;
  }
  BT_LAUNCH(mha64_fwd_kernel<false>, dim3(nqt, H, bs), dim3(M64_THREADS), M64_SMEM, s, 1, tq, tkv, p);
  return BT_OK;
}

}  // namespace bt

// Test hook: the four-CTAs-per-SM MHA on (1) / off (0) for the launches it
// serves, -1 back to the BT_MHA64 policy.
extern "C" int bt_debug_mha64(int mode) {
  BT_REQUIRE(mode >= -1 && mode <= 1, BT_ECONFIG, "bt_debug_mha64: mode -1..1");
  bt::g_mha64_override = mode;
  return BT_OK;
}
