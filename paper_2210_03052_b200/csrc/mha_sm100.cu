// Fused variable-length multi-head attention on tcgen05 (paper section III-E,
// reference attention.py:177-314).  Both kernels index the packed [T, 3k]
// QKV tensor through seq_starts and never touch a padded token.
//
// One CTA = (q-tile of 128 rows, head, sequence): work is sized by each
// sequence's true length (the grouped-problem view of the long path) and
// q tiles past a sequence's end exit immediately.  Thread t of the softmax
// warps owns query row t of the tile == TMEM lane t, so row max / row sum
// are thread-local (no shuffles) and the softmax reads S straight out of
// TMEM; P never goes to HBM.  See mha_fwd_kernel for the two paths.
//
// Q/K/V biases are already applied by the QKV GEMM epilogue.  d = 64.

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "ptx.cuh"
#include "tma_host.cuh"

namespace bt {

constexpr int MHA_D = 64;
constexpr int MHA_QT = 128;                  // query rows per CTA (UMMA M)
constexpr int MHA_KB = 128;                  // keys per block (UMMA N of S)
constexpr uint32_t MHA_TILE = 128 * 128;     // bytes of one 128 x 64 bf16 tile
constexpr int MHA_SHORT_MAX_KEYS = 384;      // TMEM: 384 S columns + 64 O columns <= 512

// Debug trace (a -DBT_TRACE_ON build with a buffer installed by
// bt_debug_mha_trace): 32 u64
// globaltimer stamps per CTA, CTA index = linear block id.
//   [0] prologue done  [1] Q landed (MMA warp)  [2+2t] S(t) ready (softmax)
//   [3+2t] item t done (softmax)  [30] O ready  [31] output stored
//   item t < 3: [16+4t] S in registers  [17+4t] max done  [18+4t] P V(t-1) done  [19+4t] P written
__device__ unsigned long long* g_mha_trace = nullptr;
// (compiled in only with -DBT_TRACE_ON, as the GEMM's: scripts/mha_trace.py
// builds that variant; the pointer check is a global load per trace point)
#ifdef BT_TRACE_ON
#define MHA_TRACE(slot)                                                                                   \
  do {                                                                                                    \
    if (g_mha_trace && (slot) < 32) {                                                                     \
      unsigned long long _t;                                                                              \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));                                              \
      g_mha_trace[((blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) * 32 + (slot)] = _t;   \
    }                                                                                                     \
  } while (0)
#else
#define MHA_TRACE(slot) \
  do {                  \
  } while (0)
#endif

struct MhaParams {
  const int32_t* seq_starts;
  __nv_bfloat16* out;
  int hidden;      // H * d
  float sl2;       // softmax scale * log2(e)
  int padded;      // 1: padded layout (reference mha_baseline, attention.py:135-174)
  int mx;          // max_seq_len (row stride of a sequence in the padded layout)
  int qg;          // query tiles per CTA (kernels with a separate output staging tile)
  const int2* sched;  // optional (packed layout): CTA z -> (start row, length), longest first
  // optional (LOOP kernels, packed layout): the tile list of bt_plan_sched --
  // *nunits query-tile units {start row, qt << 20 | length}, longest
  // sequences first; item i = (unit i / H, head i % H).  CTA c of the 1-D grid
  // starts on item c and then claims items G, G+1, ... from queue[0] as it
  // nears the end of each tile (greedy longest-first list scheduling);
  // queue[1] counts finished CTAs, the last one resets both to 0.
  const int2* units;
  const int* nunits;
  int* queue;
  int heads;
  // optional (segment kernel, packed layout): *nsegs work items of
  // bt_plan_sched, two int4 each: {key row, key end, query row, query end},
  // {first sequence, last sequence}; T = packed rows
  const int4* segs;
  const int* nsegs;
  int T;
  // optional: the instrumented FlopCounter's "mha" slot (reference
  // attention.py:232-236) -- every tile adds the work it did, 4 * d FLOPs
  // per (query row, key of its own problem)
  unsigned long long* flops;
};

// One query tile of work: rows [s0 + q0, s0 + min(q0 + 128, len)) of head h,
// keys [s0, s0 + len).
struct MhaTile {
  int s0, len, h, q0;  // keys [s0, s0 + len); query rows start at s0 + q0 (sequence tiles)
};

// Tile-list ring entry: (tile ordinal & 0xFF) << 24 | item (0xFFFFFF: none left).
constexpr uint32_t MHA_RING_NONE = 0xFFFFFFu;

// Tie a register array to a preceding tcgen05.wait::ld.
__device__ __forceinline__ void reg_tie(uint32_t (&r)[32]) {
  asm volatile(""
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                 "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]),
                 "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]),
                 "+r"(r[29]), "+r"(r[30]), "+r"(r[31]));
}

// ============================================================ kernel
// One template serves both reference paths:
//   RESIDENT = true   short path (attention.py:177-237): every K/V block of the
//                     sequence-head is TMA-staged up front and stays in shared
//                     memory (<= NST*128 keys): the tile-resident kernel.
//   RESIDENT = false  long path (attention.py:240-296): 128-key K/V blocks
//                     stream through an NST-deep TMA ring; work per CTA is the
//                     sequence's true length (grouped problem sizes).
// Softmax: single pass, online, with a lazily moved reference max.  For each
// 128-key block the two softmax threads of a query row (lanes i and i + 16 of
// one warp, 64 keys each) load their S values from TMEM ONCE into registers
// and release the S columns at once, so the MMA warp computes the next block's
// S while this block's exponentials run.  P = 2^((s - m_ref) * scale * log2 e)
// is computed into registers, then -- once the previous block's P V is done --
// written to TMEM as bf16 pairs, the A operand of O += P V (FA4-style: P never
// touches shared memory).  m_ref only moves when the row max exceeds it by
// more than 2^8 in P units; then the thread rescales its O columns in TMEM
// (ld / scale / st) and its running sum.  O / l is exact for any reference
// point, so this is the reference's long-path algorithm -- per-128-column tile
// partial (max, sum) combined by a full reduction, then exp on load
// (tensor.py:166-173, attention.py:104-122, grouped.py:202-206) -- with P
// never reaching HBM.  BT_MHA_POLY of every 16 exponentials run as a
// polynomial on the FMA pipe (ex2_poly2) so the SFU (16 ex2 / clk / SM) is not
// the only exponential pipe.  Keys past the sequence end are masked (p = 0).
//
// Warp roles (384 threads): warps 0-7 softmax / epilogue (16 query rows each,
// two threads per row), warp 8 TMA producer, warp 9 MMA issuer, warps 10-11
// idle (they complete warpgroup 2 for setmaxnreg); both issuer warps walk
// their loops warp-uniformly and issue through elect.sync.  TMEM: S [0,128)
// fp32, P [128,192) bf16 pairs, O [192,256) fp32 -> 256 columns; ~80-112 KB
// smem -> two CTAs per SM, whose latency chains interleave.
template <bool RESIDENT, int NST, bool MULTI, bool SEG = false>
struct MhaCfg {
  // MULTI (NST == 2 only: no room next to 2 CTAs per SM otherwise): a
  // separate output staging tile, so a CTA can loop over several query tiles
  // (the next Q is loaded while this tile's output is stored).  Otherwise one
  // query tile per CTA, output staged in the Q tile.
  static constexpr bool LOOP = MULTI && NST == 2;
  static constexpr uint32_t Q_OFF = 0;
  static constexpr uint32_t KV_OFF = MHA_TILE;                       // slot s: K at +32K*s, V at +32K*s+16K
  static constexpr uint32_t OUT_OFF = KV_OFF + NST * 2 * MHA_TILE;   // output staging (LOOP) else == Q
  static constexpr uint32_t BAR_OFF = OUT_OFF + (LOOP ? MHA_TILE : 0);
  static constexpr size_t SMEM = BAR_OFF + 256;
};

#ifndef BT_MHA_POLY
#define BT_MHA_POLY 2  // of every 16 exponentials, this many run as ex2_poly2 on the FMA pipe (measured 0..8: 2 best)
#endif
constexpr float MHA_RESCALE_LOG2 = 8.0f;  // move m_ref once P would exceed 2^8
// 384 threads x 2 CTAs/SM -> 80 registers each at launch (30720 per CTA).
// The issuing warpgroup drops to 32 and the two softmax warpgroups rise to
// 104 (256 x 104 + 128 x 32 = 30720): a thread holds 64 S values.
constexpr int MHA_THREADS = 384;
constexpr int MHA_REGS_ISSUE = 32;
constexpr int MHA_REGS_SOFTMAX = 104;

// SEG = true: the segment kernel.  A CTA (grid: head x item) takes one
// bt_plan_sched segment: a query tile of a sequence longer than 128 rows,
// or a group of adjacent short sequences whose rows fit one 128-row tile --
// their keys are one block, each row masked to its own sequence.  Short
// sequences then share CTAs instead of taking one each.
template <bool RESIDENT, int NST, bool MULTI, bool SEG = false>
__global__ void __launch_bounds__(MHA_THREADS, 2) mha_fwd_kernel(const __grid_constant__ CUtensorMap tm,
                                                                 const MhaParams p) {
  using Cfg = MhaCfg<RESIDENT, NST, MULTI>;
  const bool list = Cfg::LOOP && p.units != nullptr;  // tile list with a claim queue (grid-uniform)
  int h = blockIdx.y, b = blockIdx.z;
  int sb = 0, len = 0, qt0 = 0, nqt = 0, nitems = 0;
  int seg_a = 0, seg_b = 0;  // SEG: first / last sequence of the segment
  int seg_q = 0, seg_rows = 0;  // SEG: first query row, query rows
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sQ = smem + Cfg::Q_OFF;
  uint8_t* sKV = smem + Cfg::KV_OFF;
  uint8_t* sOut = smem + (Cfg::LOOP ? Cfg::OUT_OFF : Cfg::Q_OFF);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::BAR_OFF);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;         // [NST] K block landed
  uint64_t* kv_empty = bars + 1 + NST;  // [NST] K of the slot's block read by its S MMAs
  uint64_t* s_full = bars + 1 + 2 * NST;  // S(j) in TMEM
  uint64_t* s_read = s_full + 1;          // softmax has S(j) in registers: S columns free
  uint64_t* p_full = s_full + 2;          // P(j) in TMEM, O rescaled: issue P(j) V(j)
  uint64_t* pv_done = s_full + 3;         // P(j) V(j) accumulated into O: P columns free
  uint64_t* v_full = s_full + 4;          // [NST] V block landed (S(j) needs only K(j))
  uint64_t* q_empty = v_full + NST;       // the tile's last S MMA has read Q
  uint64_t* o_free = q_empty + 1;         // the softmax warps have read O (next tile may overwrite it)
  uint64_t* v_empty = o_free + 1;         // [NST] V of the slot's block read by its P V MMAs
  uint32_t* holder = reinterpret_cast<uint32_t*>(v_empty + NST);
  // [4] tile-list items of tiles t (slot t & 3), tagged with t; one word per
  // entry, written / polled with shared-memory atomics (a self-contained
  // handoff: readers use nothing else the writer stored)
  uint32_t* ring = holder + 1;

  // ---- prologue (touches no data of the previous kernels): barriers, TMEM
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    ptx::prefetch_tmap(&tm);
    ptx::mbar_init(q_full, 1);
    for (int i = 0; i < NST; ++i) {
      ptx::mbar_init(&kv_full[i], 1);
      ptx::mbar_init(&kv_empty[i], 1);
      ptx::mbar_init(&v_full[i], 1);
      ptx::mbar_init(&v_empty[i], 1);
    }
    ptx::mbar_init(s_full, 1);
    ptx::mbar_init(s_read, 256);
    ptx::mbar_init(p_full, 256);
    ptx::mbar_init(pv_done, 1);
    ptx::mbar_init(q_empty, 1);
    ptx::mbar_init(o_free, 256);
    for (int i = 0; i < 4; ++i) ring[i] = 0xFFFFFFFFu;  // tag 0xFF: no tile yet
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
  // TMEM columns: S [0,128) fp32; P [128,192) = 128 keys as packed bf16 pairs,
  // the A operand of P V (FA4-style: P never touches shared memory, which
  // would otherwise carry 64 KB of extra traffic per block); O [192,256)
  constexpr uint32_t S_COL = 0, P_COL = 128, O_COL = 192;
  ptx::griddep_launch_dependents();
  if (threadIdx.x == 0) MHA_TRACE(0);
  // The work description (seq_starts, the bt_plan_sched schedule / segments /
  // tile list) may come from an earlier kernel of the same stream (the
  // forward's plan launch): PDL only orders this kernel after its immediate
  // predecessor, so every read of it comes after griddepcontrol.wait (which
  // returns once the predecessor -- and transitively, everything it waited
  // for -- has completed and flushed).
  ptx::griddep_wait();
  bool active = true;
  if (SEG) {
    if (static_cast<int>(blockIdx.y) >= __ldg(p.nsegs)) {
      active = false;  // CTA-uniform: past the item list
    } else {
      h = blockIdx.x;
      const int4 e = __ldg(p.segs + 2 * blockIdx.y), f = __ldg(p.segs + 2 * blockIdx.y + 1);
      sb = e.x;
      len = e.y - e.x;
      seg_q = e.z;
      seg_rows = e.w - e.z;
      seg_a = f.x;
      seg_b = f.y;
    }
  } else if (list) {
    nitems = __ldg(p.nunits) * p.heads;
    if (static_cast<int>(blockIdx.x) >= nitems) active = false;  // CTA-uniform: fewer items than CTAs
    nqt = 0x7FFFFFFF;  // tiles come from the queue until it runs dry
  } else {
    if (p.sched) {  // longest problems first (plan_sched_kernel)
      const int2 e = __ldg(p.sched + b);
      sb = e.x;
      len = e.y;
    } else {
      sb = __ldg(p.seq_starts + b);
      len = __ldg(p.seq_starts + b + 1) - sb;
    }
  }
  // Packed layout: the sequence's rows start at seq_starts[b] and only its
  // len rows / keys are touched.  Padded layout (the reference's unfused
  // baseline): rows start at b*mx and the whole mx x mx rectangle is
  // computed, keys >= len masked out of the softmax (exp -> 0, the -1e9 mask
  // of attention.py:162-163) and query rows >= len written as zeros.
  const int cta_s0 = p.padded ? b * p.mx : sb;
  const int cta_work = p.padded ? p.mx : len;
  if (SEG) {
    nqt = 1;
  } else if (!list) {
    // this CTA's query tiles: qt0, qt0 + 1, ... (p.qg per CTA when Cfg::LOOP)
    const int qg = Cfg::LOOP ? p.qg : 1;
    qt0 = blockIdx.x * qg;
    if (qt0 * MHA_QT >= cta_work) active = false;  // CTA-uniform: past the sequence
    nqt = Cfg::LOOP ? min(qg, (cta_work + MHA_QT - 1) / MHA_QT - qt0) : 1;
  }
  // tile-list item -> query tile (len 0: none left)
  auto tile_of = [&](uint32_t item) -> MhaTile {
    if (item == MHA_RING_NONE) return MhaTile{0, 0, 0, 0};
    const int i = static_cast<int>(item);
    const int u = i / p.heads;
    const int2 e = __ldg(p.units + u);
    return MhaTile{e.x, e.y & 0xFFFFF, i - u * p.heads, (e.y >> 20) * MHA_QT};
  };

  // the t-th query tile of this CTA (tile list: wait for the producer's entry)
  auto tile_at = [&](int t) -> MhaTile {
    if (list) {
      uint32_t v;
      while (((v = atomicAdd(ring + (t & 3), 0u)) >> 24) != (static_cast<uint32_t>(t) & 0xFFu)) {
      }
      return tile_of(v & 0xFFFFFFu);
    }
    if (SEG) return MhaTile{cta_s0, cta_work, h, seg_q - cta_s0};
    return MhaTile{cta_s0, cta_work, h, (qt0 + t) * MHA_QT};
  };

  if (!active) {
    // nothing to do: straight to the teardown
  } else if (warp >= 8) {
    ptx::setmaxnreg_dec<MHA_REGS_ISSUE>();  // warpgroup 2: TMA (warp 8), MMA (warp 9), 2 idle warps
  if (warp == 8) {
    // ------------------------------------------------ TMA producer
    ptx::griddep_wait();  // qkv is produced by the previous kernel
    // K blocks on their own barriers ahead of V: S(j) = Q K(j)^T can start
    // before V(j) (needed only by P(j) V(j)) has landed
    int s0 = 0;
    auto load_k = [&](int j, int slot) {
      if (ptx::elect_one()) {
        ptx::mbar_arrive_expect_tx(&kv_full[slot], MHA_TILE);
        ptx::tma_load_2d(sKV + slot * 2 * MHA_TILE, &tm, &kv_full[slot], p.hidden + h * MHA_D, s0 + j * MHA_KB);
      }
      __syncwarp();
    };
    auto load_v = [&](int j, int slot) {
      if (ptx::elect_one()) {
        ptx::mbar_arrive_expect_tx(&v_full[slot], MHA_TILE);
        ptx::tma_load_2d(sKV + slot * 2 * MHA_TILE + MHA_TILE, &tm, &v_full[slot], 2 * p.hidden + h * MHA_D,
                         s0 + j * MHA_KB);
      }
      __syncwarp();
    };
    int kvg = 0;  // K/V blocks loaded so far (ring position across query tiles)
    for (int t = 0; t < nqt; ++t) {
      MhaTile it;
      if (list) {
        // claim the next item once the softmax has finished the previous
        // tile's exponentials (its P V and store remain, ~the Q load + first
        // S of the next tile): greedy list scheduling without claiming work
        // long before this CTA can start it
        uint32_t item = blockIdx.x;
        if (t > 0) {
          ptx::mbar_wait(p_full, (kvg - 1) & 1);  // kvg = blocks of the previous tiles
          ptx::mbar_wait(q_empty, (t - 1) & 1);
          if (lane == 0) item = gridDim.x + atomicAdd(p.queue, 1);
          item = __shfl_sync(0xffffffffu, item, 0);
          if (item >= static_cast<uint32_t>(nitems)) item = MHA_RING_NONE;
        }
        if (lane == 0) atomicExch(ring + (t & 3), (static_cast<uint32_t>(t) & 0xFFu) << 24 | item);
        __syncwarp();
        if (item == MHA_RING_NONE) break;
        it = tile_of(item);
      } else {
        if (t > 0) ptx::mbar_wait(q_empty, (t - 1) & 1);  // the previous tile's S MMAs are done with sQ
        it = tile_at(t);
      }
      s0 = it.s0;
      h = it.h;
      const int nkb = (it.len + MHA_KB - 1) / MHA_KB;
      if (ptx::elect_one()) {
        ptx::mbar_arrive_expect_tx(q_full, MHA_TILE);
        ptx::tma_load_2d(sQ, &tm, q_full, h * MHA_D, s0 + it.q0);
      }
      __syncwarp();
      if (RESIDENT) {
        if (t == 0) {  // K / V stay resident for every query tile of the CTA
          for (int j = 0; j < nkb; ++j) load_k(j, j);
          for (int j = 0; j < nkb; ++j) load_v(j, j);
        }
      } else {
        for (int j = 0; j < nkb; ++j, ++kvg) {
          const int slot = kvg % NST;
          // K and V slots are released separately: K(j) once S(j) has read it,
          // V(j) once P(j) V(j) has -- the next K loads a block ahead of the
          // P V chain, so S(j + 1) is ready when the softmax releases S(j)
          ptx::mbar_wait(&kv_empty[slot], ((kvg / NST) & 1) ^ 1u);
          load_k(j, slot);
          ptx::mbar_wait(&v_empty[slot], ((kvg / NST) & 1) ^ 1u);
          load_v(j, slot);
        }
      }
    }
  } else if (warp == 9) {
    // ------------------------------------------------ MMA issuer
    constexpr uint32_t idesc_s = ptx::idesc_bf16(128, MHA_KB, false, false);  // Q K^T, both K-major
    constexpr uint32_t idesc_o = ptx::idesc_bf16(128, MHA_D, false, true);    // P (TMEM, K-major) x V (MN-major)
    const uint64_t q_desc = ptx::sdesc_sw128(ptx::smem_u32(sQ), 1024, 16);
    const uint32_t kv_base = ptx::smem_u32(sKV);
    auto issue_pv = [&](int g, int jt, int t, int pslot, uint32_t kvpar, int work) {
      // O (+)= P(g) V(g): item g is block jt of query tile t; only the
      // k-steps that hold keys of the problem
      ptx::mbar_wait(&v_full[pslot], kvpar);
      ptx::mbar_wait(p_full, g & 1);
      if (jt == 0 && t > 0) ptx::mbar_wait(o_free, (t - 1) & 1);  // the previous tile's O has been read
      ptx::tc_fence_after();
      const int nks = min(MHA_KB, work - jt * MHA_KB + 15) / 16;
      const uint64_t v_desc = ptx::sdesc_sw128(kv_base + pslot * 2 * MHA_TILE + MHA_TILE, 1024, MHA_TILE);
      if (ptx::elect_one()) {
        for (int ks = 0; ks < nks; ++ks)
          ptx::mma_bf16_ts(tmem + O_COL, tmem + P_COL + 8 * ks, v_desc + ks * ((16 * 128) >> 4), idesc_o,
                           (jt > 0 || ks > 0) ? 1u : 0u);
        ptx::mma_commit(pv_done);
        if (!RESIDENT) ptx::mma_commit(&v_empty[pslot]);  // V of this block consumed
      }
      __syncwarp();
    };
    int g = 0, kvg = 0;  // items issued (S), K/V ring position
    int prev_jt = 0, prev_t = 0, prev_slot = 0, prev_work = 0;
    uint32_t prev_par = 0;
    for (int t = 0; t < nqt; ++t) {
      const int work = tile_at(t).len;
      if (work == 0) break;  // tile list ran dry
      const int nkb = (work + MHA_KB - 1) / MHA_KB;
      ptx::mbar_wait(q_full, t & 1);
      if (lane == 0 && t == 0) MHA_TRACE(1);
      for (int j = 0; j < nkb; ++j, ++g, ++kvg) {
        const int slot = RESIDENT ? j : kvg % NST;
        const uint32_t par = RESIDENT ? 0u : static_cast<uint32_t>((kvg / NST) & 1);
        ptx::mbar_wait(&kv_full[slot], par);
        if (g > 0) ptx::mbar_wait(s_read, (g - 1) & 1);  // S(g-1) is in the softmax registers
        ptx::tc_fence_after();
        const uint64_t k_desc = ptx::sdesc_sw128(kv_base + slot * 2 * MHA_TILE, 1024, 16);
        if (ptx::elect_one()) {
#pragma unroll
          for (int kk = 0; kk < MHA_D / 16; ++kk)
            ptx::mma_bf16_ss(tmem + S_COL, q_desc + 2 * kk, k_desc + 2 * kk, idesc_s, kk > 0);
          ptx::mma_commit(s_full);
          if (!RESIDENT) ptx::mma_commit(&kv_empty[slot]);  // K of this block consumed
          if (j == nkb - 1) ptx::mma_commit(q_empty);  // this tile's Q is no longer read
        }
        __syncwarp();
        if (g > 0) issue_pv(g - 1, prev_jt, prev_t, prev_slot, prev_par, prev_work);
        prev_jt = j;
        prev_t = t;
        prev_slot = slot;
        prev_par = par;
        prev_work = work;
      }
    }
    issue_pv(g - 1, prev_jt, prev_t, prev_slot, prev_par, prev_work);
  }
  } else {
    ptx::setmaxnreg_inc<MHA_REGS_SOFTMAX>();  // warpgroups 0-1: softmax
    // ------------------------------------------------ softmax: a row of S is
    // shared by two threads of ONE warp (tcgen05 .16x32bx2 accesses): warp
    // w = quarter + 4 * half owns the 16 TMEM lanes 32 * quarter + 16 * half
    // .. +15 (query rows); lane i < 16 takes keys 0-63 of each block, lane
    // i + 16 keys 64-127 of the same row.  The row max is combined with one
    // shuffle (no shared memory, no barrier between warps); row sums stay
    // per-thread partials until the end.  Warp-uniform skipping: warps whose
    // 16 query rows lie past the tile's rows.
    const int quarter = warp & 3, half = warp >> 2;
    const int kh = lane >> 4;  // chunk c of a block: keys 64c + 32kh .. + 31
    const int row0 = quarter * 32 + half * 16;
    const int row = row0 + (lane & 15);
    const uint32_t trow = tmem + (static_cast<uint32_t>(row0) << 16);
    const uint32_t s_my = trow + S_COL;  // chunk c: columns 64c (+32 for kh = 1)
    const uint32_t p_my = trow + P_COL;  // chunk c: columns 32c (+16 for kh = 1)
    const uint32_t o_my = trow + O_COL;  // columns 0-31 (+32 for kh = 1)
    const float sl2 = p.sl2;
    int g = 0;  // items consumed, across query tiles
    for (int t = 0; t < nqt; ++t) {
    const MhaTile it = tile_at(t);
    if (it.len == 0) break;  // tile list ran dry
    const int q0 = it.q0, s0 = it.s0, work = it.len, hh = it.h;
    if (list) len = it.len;
    const int nkb = (work + MHA_KB - 1) / MHA_KB;
    // query rows of this tile that exist (sequence tiles: inside the
    // sequence; segments: the segment's rows)
    const int rows_here = SEG ? seg_rows : work - q0;
    const bool warp_live = row0 < rows_here;
    // SEG: my row's keys [ks, ke) relative to s0 (its own sequence)
    int ks = 0, ke = len;
    if (SEG && seg_a < seg_b) {  // a group of short sequences
      const int r = s0 + q0 + row;
      if (row < rows_here) {
        int lo = seg_a, hi = seg_b;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (__ldg(p.seq_starts + mid) <= r) lo = mid; else hi = mid - 1;
        }
        ks = __ldg(p.seq_starts + lo) - s0;
        ke = __ldg(p.seq_starts + lo + 1) - s0;
      } else {
        ks = ke = 0;
      }
    }
    float mref = -INFINITY, lsum = 0.f;
    for (int j = 0; j < nkb; ++j, ++g) {
      const int kblk = min(MHA_KB, len - j * MHA_KB);  // keys of the problem in this block
      // my keys of chunk c are 64c + 32kh + i (i < 32): valid iff i < kblk - 64c - 32kh
      // (SEG: my row's own sequence's keys, 64c + 32kh + i in [ks, ke) - j*128)
      const int kof = j * MHA_KB + kh * 32;
      ptx::mbar_wait(s_full, g & 1);
      ptx::tc_fence_after();
      if (threadIdx.x == 0 && t == 0) MHA_TRACE(2 + 2 * j);
      uint32_t r0[32], r1[32];  // my 64 S values of this row: chunk 0, chunk 1
      if (warp_live) {
        ptx::tmem_ld_16x2_32<32>(s_my, r0);
        ptx::tmem_ld_16x2_32<32>(s_my + 64, r1);
        ptx::tmem_wait_ld(r0);
        reg_tie(r1);
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(s_read);  // S is in registers: the MMA warp may overwrite it with the next block
      if (threadIdx.x == 0 && t == 0 && j < 3) MHA_TRACE(16 + 4 * j);
      // keys outside the problem (past its end; SEG: outside my row's own
      // sequence) -> s = -inf: out of the max, exp -> exactly 0
      auto mask = [&](uint32_t (&r)[32], int c) {
        const int lo = SEG ? ks - kof - 64 * c : 0;
        const int hi = (SEG ? ke : len) - kof - 64 * c;
        if (lo > 0 || hi < 32) {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (i < lo || i >= hi) r[i] = 0xff800000u;
        }
      };
      bool need = false;
      float alpha = 1.f;
      if (warp_live) {
        mask(r0, 0);
        mask(r1, 1);
        float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          m4[0] = ptx::max3(m4[0], __uint_as_float(r0[i]), __uint_as_float(r0[i + 1]));
          m4[1] = ptx::max3(m4[1], __uint_as_float(r0[i + 2]), __uint_as_float(r0[i + 3]));
          m4[2] = ptx::max3(m4[2], __uint_as_float(r1[i]), __uint_as_float(r1[i + 1]));
          m4[3] = ptx::max3(m4[3], __uint_as_float(r1[i + 2]), __uint_as_float(r1[i + 3]));
        }
        // the row's other half is lane ^ 16 of this warp
        const float mloc = fmaxf(ptx::max3(m4[0], m4[1], m4[2]), m4[3]);
        const float bmax = fmaxf(mloc, __shfl_xor_sync(0xffffffffu, mloc, 16));
        const float mnew = fmaxf(mref, bmax);
        need = (mnew - mref) * sl2 > MHA_RESCALE_LOG2;  // true on the first block (mref = -inf)
        alpha = (need && mref != -INFINITY) ? ptx::ex2_approx((mref - mnew) * sl2) : 1.f;
        if (need) mref = mnew;
        if (threadIdx.x == 0 && t == 0 && j < 3) MHA_TRACE(17 + 4 * j);
      }
      // P = 2^((s - m_ref) * scale * log2 e): BT_MHA_POLY of every 16 on the
      // FMA pipe, the rest on the SFU.  (SEG: a row whose sequence has no key
      // in the blocks so far keeps m_ref = -inf; its S are all -inf, so any
      // finite offset gives P = 0)
      const float msc = (SEG && mref == -INFINITY) ? 0.f : mref * sl2;
      const unsigned long long sl2x2 = ptx::f2(sl2, sl2), nm2 = ptx::f2(-msc, -msc);
      unsigned long long sum4[4] = {0ull, 0ull, 0ull, 0ull};  // 4 independent add chains
      auto exps = [&](const uint32_t (&r)[32], uint32_t (&pp)[16]) {
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          float x0, x1, e0, e1;
          ptx::unf2(ptx::fma2(ptx::f2(__uint_as_float(r[i]), __uint_as_float(r[i + 1])), sl2x2, nm2), x0, x1);
          if ((i & 15) < BT_MHA_POLY) {
            ptx::ex2_poly2(x0, x1, e0, e1);  // masked key (x = -inf): exactly 0
          } else {
            e0 = ptx::ex2_approx(x0);  // ex2(-inf) = 0
            e1 = ptx::ex2_approx(x1);
          }
          sum4[(i >> 1) & 3] = ptx::add2(sum4[(i >> 1) & 3], ptx::f2(e0, e1));
          pp[i / 2] = ptx::pack_bf16x2(e0, e1);
        }
      };
      if (j > 0) {
        ptx::mbar_wait(pv_done, (g - 1) & 1);  // P(g-1) V(g-1) is in O; the P columns are free
        ptx::tc_fence_after();
      }
      if (threadIdx.x == 0 && t == 0 && j < 3) MHA_TRACE(18 + 4 * j);
      if (warp_live) {
        uint32_t pp[16];  // my 32 keys of chunk c as bf16 pairs -> P columns 32c (+16 for kh = 1)
        exps(r0, pp);
        ptx::tmem_st_16x2_16<16>(p_my, pp);
        if (64 >= kblk) {
          // CTA-uniform: no key of the problem among keys 64-127 -> P = 0
          // (stored from zero registers on this path of its own, so pp is
          // never half-assigned and stays in registers)
          ptx::tmem_st_16x2_16_zero<16>(p_my + 32);
        } else {
          exps(r1, pp);
          ptx::tmem_st_16x2_16<16>(p_my + 32, pp);
        }
      }

      if (warp_live) {
        const unsigned long long bsum2 = ptx::add2(ptx::add2(sum4[0], sum4[1]), ptx::add2(sum4[2], sum4[3]));
        float s0f, s1f;
        ptx::unf2(bsum2, s0f, s1f);
        lsum = lsum * alpha + (s0f + s1f);  // my keys' partial row sum
        if (__any_sync(0xffffffffu, need && j > 0)) {
          // the reference max moved (rare): my 32 O columns *= 2^((m_old - m_new) * scale)
          const unsigned long long a2 = ptx::f2(alpha, alpha);
          uint32_t o[32];
          ptx::tmem_ld_16x2_32<32>(o_my, o);
          ptx::tmem_wait_ld(o);
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            float a, c;
            ptx::unf2(ptx::mul2(ptx::f2(__uint_as_float(o[i]), __uint_as_float(o[i + 1])), a2), a, c);
            o[i] = __float_as_uint(a);
            o[i + 1] = __float_as_uint(c);
          }
          ptx::tmem_st_16x2_32<32>(o_my, o);
        }
        ptx::tmem_wait_st();
      }
      if (threadIdx.x == 0 && t == 0 && j < 3) MHA_TRACE(19 + 4 * j);
      ptx::tc_fence_before();
      ptx::mbar_arrive(p_full);
      if (threadIdx.x == 0 && t == 0) MHA_TRACE(3 + 2 * j);
    }
    ptx::mbar_wait(pv_done, (g - 1) & 1);  // this tile's last P V
    ptx::tc_fence_after();
    if (threadIdx.x == 0 && t == 0) MHA_TRACE(30);
    // O / l -> bf16 rows staged in shared memory -> coalesced 16-byte stores,
    // 4 rows per warp instruction; a warp stages and stores its own 16 rows
    if (warp_live) {
      uint32_t o[32];
      ptx::tmem_ld_16x2_32<32>(o_my, o);
      const float l = lsum + __shfl_xor_sync(0xffffffffu, lsum, 16);
      ptx::tmem_wait_ld(o);
      const float inv = (SEG ? row < rows_here : q0 + row < len) ? 1.0f / l : 0.f;
      const unsigned long long inv2 = ptx::f2(inv, inv);
      uint8_t* mine = sOut + row * 128;
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        uint32_t w[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float a, b2;
          ptx::unf2(ptx::mul2(ptx::f2(__uint_as_float(o[8 * jj + 2 * e]), __uint_as_float(o[8 * jj + 2 * e + 1])), inv2),
                    a, b2);
          w[e] = ptx::pack_bf16x2(a, b2);
        }
        const int chunk = kh * 4 + jj;
        *reinterpret_cast<uint4*>(mine + ((chunk ^ (row & 7)) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
      }
      __syncwarp();  // the warp's 16 rows are staged
      ptx::griddep_wait();  // out may still be read by the previous kernel
      // lane -> (row of the warp's 16, 16 B chunk)
#pragma unroll
      for (int it = 0; it < 4; ++it) {
        const int rr = row0 + it * 4 + (lane >> 3);
        const int jj = lane & 7;
        if (rr < rows_here) {
          const uint4 v = *reinterpret_cast<const uint4*>(sOut + rr * 128 + ((jj ^ (rr & 7)) << 4));
          *reinterpret_cast<uint4*>(p.out + static_cast<size_t>(s0 + q0 + rr) * p.hidden + hh * MHA_D + jj * 8) = v;
        }
      }
      if (list || t + 1 < nqt) __syncwarp();  // the warp's rows are stored: sOut free for the next tile
    }
    if (p.flops != nullptr && warp_live) {
      // instrumentation: the key-half-0 thread of each row counts the row's keys
      // (padded mode computes the whole mx x mx rectangle, reference mha_baseline)
      const unsigned keys = (kh == 0 && row < rows_here) ? static_cast<unsigned>(p.padded ? work : ke - ks) : 0u;
      const unsigned w = __reduce_add_sync(0xffffffffu, keys);
      if (lane == 0 && w) atomicAdd(p.flops, 4ull * MHA_D * w);
    }
    if (threadIdx.x == 0 && (t == 1 || t == 2)) MHA_TRACE(27 + t);  // tiles 1, 2 stored (slots 28, 29)
    if (list || t + 1 < nqt) {
      ptx::tc_fence_before();
      ptx::mbar_arrive(o_free);  // O of this tile has been read: the next tile's first P V may overwrite it
    }
    }  // query tiles
    if (threadIdx.x == 0) MHA_TRACE(31);
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 256);
  }
  if (list && active && threadIdx.x == 0) {
    // every claim of this CTA precedes this point; the last CTA resets the
    // queue for the next launch
    const int participants = min(static_cast<int>(gridDim.x), nitems);
    __threadfence();
    if (atomicAdd(p.queue + 1, 1) == participants - 1) {
      p.queue[0] = 0;
      p.queue[1] = 0;
      __threadfence();
    }
  }
}

template <typename K>
static int set_smem(K kern, size_t bytes) {
  BT_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
  // two CTAs per SM: the multi-tile kernels need 2 x 99 KB, more than the
  // default carveout leaves for shared memory
  BT_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  return BT_OK;
}

// Query tiles per CTA: BT_MHA_QG (1..8) or bt_debug_mha_qg override the
// policy (A/B measurement, tests).
static int g_mha_qg_override = 0;
static int mha_qtiles_per_cta(int nqt, bool many_waves) {
  static int forced = -1;
  if (forced < 0) {
    const char* e = getenv("BT_MHA_QG");
    forced = (e && e[0] >= '1' && e[0] <= '8') ? e[0] - '0' : 0;
  }
  const int qg = g_mha_qg_override ? g_mha_qg_override : forced ? forced : (many_waves ? 4 : 1);
  return qg < nqt ? qg : nqt;
}

// Tile-list policy: BT_MHA_LIST=0 disables it (A/B measurement);
// bt_debug_mha_list overrides (0 off, 1 automatic, 2 always) and can pin the
// grid size (tests: many claims per CTA on a small batch).
static int g_mha_list_mode = -1, g_mha_list_grid = 0, g_mha_seg_mode = -1;
// Segment-kernel policy (batches of bs <= 256, max_seq_len <= 256):
// BT_MHA_SEG=0 disables it, 2 forces it in its domain; bt_debug_mha_seg
// overrides (0 off, 1 by size, 2 forced).
static int mha_seg_mode() {
  if (g_mha_seg_mode >= 0) return g_mha_seg_mode;
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("BT_MHA_SEG");
    env = (e && (e[0] == '0' || e[0] == '2')) ? e[0] - '0' : 1;
  }
  return env;
}
static int mha_list_mode() {
  if (g_mha_list_mode >= 0) return g_mha_list_mode;
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("BT_MHA_LIST");
    env = (e && e[0] == '0') ? 0 : 1;
  }
  return env;
}

// Instrumented FLOP counting (bt_flops_enable): device counter the MHA
// tiles add their work to, null when off.
unsigned long long* g_mha_flops = nullptr;

bool mha64_enabled();
int mha64_set_trace(unsigned long long* buf);
int mha64_launch(const void* qkv, const int32_t* seq_starts, const void* sched, int bs, int mx, int H, int T,
                 void* out, cudaStream_t s);

int mha_launch(const void* qkv, const int32_t* seq_starts, int bs, int mx, int H, int d, int cutoff, int T,
               void* out, int force_path, cudaStream_t s, int padded, const void* sched) {
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
  p.padded = padded;
  p.mx = mx;
  p.sched = padded ? nullptr : static_cast<const int2*>(sched);
  p.qg = 1;
  p.units = nullptr;
  p.nunits = nullptr;
  p.queue = nullptr;
  p.segs = nullptr;
  p.nsegs = nullptr;
  p.T = T;
  p.heads = H;
  p.flops = g_mha_flops;
  BT_REQUIRE(!padded || T == bs * mx, BT_ESHAPE, "padded mha: qkv must have bs*mx = %d rows, got %d", bs * mx, T);
  const int nqt = (mx + MHA_QT - 1) / MHA_QT;
  // dispatch_mha rule (attention.py:309-314); the resident (short) kernel
  // holds at most 384 keys on chip.
  bool use_short = mx <= cutoff && mx <= MHA_SHORT_MAX_KEYS;
  if (force_path == 1) use_short = true;
  if (force_path == 2) use_short = false;
  BT_REQUIRE(!use_short || mx <= MHA_SHORT_MAX_KEYS, BT_ECONFIG, "short MHA holds <= 384 keys, mx=%d", mx);
  // Query tiles per CTA: with many waves of CTAs (large batches) a CTA walks
  // all tiles of its sequence-head, sharing K / V and overlapping the next
  // tile's Q load with the previous tile's output store; with few waves the
  // longer per-CTA chain would cost more than that saves, so one tile per CTA.
  const int sms = num_sms() > 0 ? num_sms() : 148;
  const long long ctas1 = static_cast<long long>(nqt) * H * bs;
  // Tile list (bt_plan_sched's units): for launches of many waves a fixed
  // grid of slot-many CTAs (2 per SM) claims query tiles longest-first from a
  // queue; each CTA's next Q load overlaps its previous tile's output store
  // and the per-CTA set-up is paid once.  Measured at C5 (BERT-large, 2048 x
  // 512): 2806 vs 2917 us per launch against 4 consecutive tiles per CTA.
  // Few waves (C2, C3) keep one tile per CTA: there the multi-tile kernel's
  // longer per-tile chain (its issuer warps spill at 32 registers) costs more
  // than the balance gains (C2 13.9 vs 10.7 us, C3 26.6 vs 26.1 us).
  // Segment kernel (short batches): adjacent short sequences share a CTA.
  // Mode 1 keeps it where it measured faster than the four-CTA kernel: launches
  // of about one wave (C2 16 x 256: 8.1 vs 12.0 us in the graph) and
  // max_seq_len <= 64, where it packs several sequences per query tile
  // (64 x 64: 8.4 vs 9.1 us); beyond that the four-CTA kernel wins (32 x 256:
  // 13.7 vs 15.6, 256 x 256: 71.5 vs 106.8, 256 x 128: 35.5 vs 48.6 us;
  // scripts/mha_time.py).  Mode 2 forces it inside its domain.
  const int seg_mode = mha_seg_mode();
  const bool m64 = !padded && mha64_enabled();
  const bool seg_small = !m64 || mx <= 64 || ctas1 <= 3LL * sms;
  if (p.sched && bs <= SEG_MAX_BS && mx <= SEG_MAX_MX && (seg_mode == 2 || (seg_mode == 1 && seg_small))) {
    p.nsegs = reinterpret_cast<const int*>(static_cast<const uint8_t*>(sched) + sched_segs_offset(bs, mx));
    p.segs = reinterpret_cast<const int4*>(p.nsegs + 4);
    static bool set = false;
    if (!set) {
      BT_TRY(set_smem(mha_fwd_kernel<false, 2, false, true>, MhaCfg<false, 2, false>::SMEM));
      set = true;
    }
    BT_LAUNCH((mha_fwd_kernel<false, 2, false, true>), dim3(H, bs * nqt), dim3(MHA_THREADS),
              MhaCfg<false, 2, false>::SMEM, s, 1, tm, p);
    return BT_OK;
  }
  // the four-CTAs-per-SM kernel (mha64_sm100.cu) for every other packed
  // launch: measured faster than both the one-tile and the tile-list modes
  // below (C3 24.5 -> 21.9 us, C5 2.84-2.96 -> 2.45-2.55 ms per launch)
  if (m64) return mha64_launch(qkv, seq_starts, p.sched, bs, mx, H, T, out, s);
  const int list_mode = mha_list_mode();
  if (p.sched && list_mode > 0) {
    static int slots = 0;
    if (slots == 0) {
      // resident CTAs per SM from the resources themselves: the occupancy
      // API reports 1 for these kernels (measured), while two run per SM
      // (per-CTA traces: 296 CTAs start within 1.2 us)
      BT_TRY(set_smem(mha_fwd_kernel<false, 2, true>, MhaCfg<false, 2, true>::SMEM));
      cudaFuncAttributes fa;
      BT_CUDA_CHECK(cudaFuncGetAttributes(&fa, mha_fwd_kernel<false, 2, true>));
      int dev = 0, sm_smem = 0, rsv = 0, sm_regs = 0;
      BT_CUDA_CHECK(cudaGetDevice(&dev));
      BT_CUDA_CHECK(cudaDeviceGetAttribute(&sm_smem, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev));
      BT_CUDA_CHECK(cudaDeviceGetAttribute(&rsv, cudaDevAttrReservedSharedMemoryPerBlock, dev));
      BT_CUDA_CHECK(cudaDeviceGetAttribute(&sm_regs, cudaDevAttrMaxRegistersPerMultiprocessor, dev));
      const int by_smem = sm_smem / static_cast<int>(MhaCfg<false, 2, true>::SMEM + rsv);
      const int by_regs = sm_regs / (MHA_THREADS * (fa.numRegs > 0 ? fa.numRegs : 80));
      const int by_tmem = 512 / 256;
      const int per_sm = std::min(std::min(by_smem, by_regs), by_tmem);
      BT_REQUIRE(per_sm >= 1, BT_ECUDA, "mha: the tile-list kernel does not fit on an SM");
      slots = per_sm * sms;
    }
    const int grid = g_mha_list_grid > 0 ? g_mha_list_grid : slots;
    if (ctas1 > 16LL * slots || list_mode == 2) {
      p.nunits = reinterpret_cast<const int*>(static_cast<const uint8_t*>(sched) + sched_units_offset(bs));
      p.units = reinterpret_cast<const int2*>(p.nunits + 4);
      p.queue = const_cast<int*>(p.nunits + 1);
      BT_LAUNCH((mha_fwd_kernel<false, 2, true>), dim3(grid), dim3(MHA_THREADS), MhaCfg<false, 2, true>::SMEM, s, 1,
                tm, p);
      return BT_OK;
    }
  }
  const int qg = mha_qtiles_per_cta(nqt, ctas1 > 16LL * 2 * sms);
  p.qg = qg;
  const dim3 grid_multi((nqt + qg - 1) / qg, H, bs), grid_one(nqt, H, bs);
#define BT_MHA_GO(R, N, M, G)                                                                                 \
  do {                                                                                                        \
    static bool set = false;                                                                                  \
    if (!set) {                                                                                               \
      BT_TRY(set_smem(mha_fwd_kernel<R, N, M>, MhaCfg<R, N, M>::SMEM));                                       \
      set = true;                                                                                             \
    }                                                                                                         \
    BT_LAUNCH((mha_fwd_kernel<R, N, M>), G, dim3(MHA_THREADS), MhaCfg<R, N, M>::SMEM, s, 1, tm, p);           \
  } while (0)
  if (use_short && mx <= 2 * MHA_KB) {
    if (qg > 1)
      BT_MHA_GO(true, 2, true, grid_multi);
    else
      BT_MHA_GO(true, 2, false, grid_one);
  } else if (use_short) {
    BT_MHA_GO(true, 3, false, grid_one);
  } else {
    if (qg > 1)
      BT_MHA_GO(false, 2, true, grid_multi);
    else
      BT_MHA_GO(false, 2, false, grid_one);
  }
#undef BT_MHA_GO
  return BT_OK;
}

}  // namespace bt

// Test hook: force the query tiles per MHA CTA (0 = automatic policy).
extern "C" int bt_debug_mha_qg(int qg) {
  BT_REQUIRE(qg >= 0 && qg <= 8, BT_ECONFIG, "bt_debug_mha_qg: 0..8");
  bt::g_mha_qg_override = qg;
  return BT_OK;
}

// Test hook: tile-list mode (0 off, 1 automatic, 2 always, -1 back
// to the BT_MHA_LIST policy) and its grid size (0 = the resident CTA slots).
extern "C" int bt_debug_mha_list(int mode, int grid) {
  BT_REQUIRE(mode >= -1 && mode <= 2 && grid >= 0, BT_ECONFIG, "bt_debug_mha_list: mode -1..2, grid >= 0");
  bt::g_mha_list_mode = mode;
  bt::g_mha_list_grid = grid;
  return BT_OK;
}

// Test hook: the segment kernel (0 off, 1 / 2 on where it applies, -1 back to
// the BT_MHA_SEG policy).
extern "C" int bt_debug_mha_seg(int mode) {
  BT_REQUIRE(mode >= -1 && mode <= 2, BT_ECONFIG, "bt_debug_mha_seg: mode -1..2");
  bt::g_mha_seg_mode = mode;
  return BT_OK;
}

extern "C" int bt_debug_mha_trace(unsigned long long* buf) {
  BT_CUDA_CHECK(cudaMemcpyToSymbol(bt::g_mha_trace, &buf, sizeof(buf)));
  return bt::mha64_set_trace(buf);  // the four-CTA kernel's trace points (mha64_sm100.cu)
}

extern "C" int bt_mha_varlen(const void* qkv, const int32_t* seq_starts, int bs, int mx, int H, int d, int cutoff,
                             int split_seq_len, void* out, int T, bt_stream_t stream) {
  BT_REQUIRE(split_seq_len >= 1, BT_ESHAPE, "split_seq_len must be >= 1, got %d", split_seq_len);
  return bt::mha_launch(qkv, seq_starts, bs, mx, H, d, cutoff, T, out, 0, bt::as_stream(stream), 0, nullptr);
}

extern "C" int bt_mha_varlen_sched(const void* qkv, const int32_t* seq_starts, const void* sched, int bs, int mx,
                                   int H, int d, int cutoff, void* out, int T, bt_stream_t stream) {
  return bt::mha_launch(qkv, seq_starts, bs, mx, H, d, cutoff, T, out, 0, bt::as_stream(stream), 0, sched);
}

extern "C" int bt_mha_padded(const void* qkv, const int32_t* seq_starts, int bs, int mx, int H, int d, void* out,
                             bt_stream_t stream) {
  return bt::mha_launch(qkv, seq_starts, bs, mx, H, d, 384, bs * mx, out, 0, bt::as_stream(stream), 1, nullptr);
}

// Test hook: force the short (1) or long (2) kernel regardless of cutoff.
extern "C" int bt_mha_varlen_path(const void* qkv, const int32_t* seq_starts, int bs, int mx, int H, int d,
                                  void* out, int T, int path, bt_stream_t stream) {
  return bt::mha_launch(qkv, seq_starts, bs, mx, H, d, 384, T, out, path, bt::as_stream(stream), 0, nullptr);
}

// Debug hook: resident CTAs per SM of the MHA variants (0: short NST 2,
// 1: short NST 3, 2: long, 3: multi-tile long); -1 on error.  Also writes
// regs / static smem / max dynamic smem of the variant into info[3].
extern "C" int bt_debug_mha_occupancy(int which, int* info) {
  auto probe = [&](auto kern, size_t smem) -> int {
    if (bt::set_smem(kern, smem) != BT_OK) return -1;
    cudaFuncAttributes a;
    if (cudaFuncGetAttributes(&a, kern) != cudaSuccess) return -1;
    if (info) {
      info[0] = a.numRegs;
      info[1] = static_cast<int>(a.sharedSizeBytes);
      info[2] = a.maxDynamicSharedSizeBytes;
    }
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, bt::MHA_THREADS, smem) != cudaSuccess) return -1;
    return n;
  };
  switch (which) {
    case 0: return probe(bt::mha_fwd_kernel<true, 2, false>, bt::MhaCfg<true, 2, false>::SMEM);
    case 1: return probe(bt::mha_fwd_kernel<true, 3, false>, bt::MhaCfg<true, 3, false>::SMEM);
    case 2: return probe(bt::mha_fwd_kernel<false, 2, false>, bt::MhaCfg<false, 2, false>::SMEM);
    case 3: return probe(bt::mha_fwd_kernel<false, 2, true>, bt::MhaCfg<false, 2, true>::SMEM);
    default: return -1;
  }
}
