// Zero-padding removal (ByteTransformer section III-D, reference packing.py):
//   * plan: mask -> lengths -> exclusive prefix sum (seq_starts) -> offsets
//   * pack: gather valid rows into a contiguous [T, k] tensor (+ fp32->bf16)
//   * unpack: scatter back with exact-zero padded rows (+ bf16->fp32)
// All kernels are HBM-bound data movement; 16-byte vector accesses, grids
// sized in multiples of the SM count.

#include <algorithm>
#include <cstdarg>
#include <cstdlib>
#include <cstring>

#include <type_traits>

#include "common.cuh"
#include "ptx.cuh"

namespace bt {

// ------------------------------------------------------------ library state
std::atomic<long long> g_launches{0};
static thread_local char t_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(t_err, sizeof(t_err), fmt, ap);
  va_end(ap);
}
const char* last_error() { return t_err; }

bool pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("BT_PDL");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on != 0;
}

int num_sms() {
  static int cached = -1;
  if (cached < 0) {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
      cudaGetLastError();
      return 0;
    }
    cached = n;
  }
  return cached;
}

// ------------------------------------------------------------------ plan
// One warp per mask row: count ones, find the first zero, flag entries that
// are not 0/1.  A row is prefix-shaped iff count == first_zero (packing.py:
// 102-109 rejects anything else).
__global__ void plan_rows_kernel(const uint8_t* __restrict__ mask, int bs, int mx, int32_t* __restrict__ lengths,
                                 int32_t* __restrict__ status) {
  ptx::griddep_launch_dependents();
  ptx::griddep_wait();
  const int warps_per_block = blockDim.x / 32;
  const int lane = threadIdx.x & 31;
  for (int row = blockIdx.x * warps_per_block + threadIdx.x / 32; row < bs; row += gridDim.x * warps_per_block) {
    const uint8_t* m = mask + static_cast<size_t>(row) * mx;
    int ones = 0, first_zero = mx, bad = 0;
    for (int j = lane; j < mx; j += 32) {
      const uint8_t v = m[j];
      bad |= (v > 1);
      ones += (v == 1);
      if (v == 0 && j < first_zero) first_zero = j;
    }
    for (int o = 16; o; o >>= 1) {
      ones += __shfl_xor_sync(0xffffffffu, ones, o);
      bad |= __shfl_xor_sync(0xffffffffu, bad, o);
      first_zero = min(first_zero, __shfl_xor_sync(0xffffffffu, first_zero, o));
    }
    if (lane == 0) {
      lengths[row] = ones;
      int st = 0;
      if (bad) st |= 1;
      if (!bad && ones != first_zero) st |= 2;
      if (ones == 0) st |= 4;
      if (st) atomicOr(status, st);
    }
  }
}

// Single-CTA exclusive scan of lengths -> seq_starts[bs+1] (+ total T).
// 1024 threads, chunked over bs with a running carry.
__device__ __forceinline__ void plan_scan_body(const int32_t* __restrict__ lengths, int bs,
                                               int32_t* __restrict__ seq_starts, int32_t* __restrict__ valid_cnt,
                                               int32_t* sm_starts = nullptr) {
  __shared__ int32_t warp_sums[32];
  __shared__ int32_t carry_s;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) carry_s = 0;
  __syncthreads();
  for (int base = 0; base < bs; base += 1024) {
    const int i = base + tid;
    const int v = (i < bs) ? lengths[i] : 0;
    int x = v;  // inclusive warp scan
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[wid] = x;
    __syncthreads();
    if (wid == 0) {
      int w = warp_sums[lane];
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      warp_sums[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    const int carry = carry_s;
    const int incl = x + (wid ? warp_sums[wid - 1] : 0) + carry;
    if (i < bs) {
      seq_starts[i] = incl - v;
      if (sm_starts) sm_starts[i] = incl - v;
    }
    __syncthreads();
    if (tid == 1023) carry_s = incl;
    __syncthreads();
  }
  if (tid == 0) {
    seq_starts[bs] = carry_s;
    if (sm_starts) sm_starts[bs] = carry_s;
    if (valid_cnt) *valid_cnt = carry_s;
  }
}

__global__ void __launch_bounds__(1024) plan_scan_kernel(const int32_t* __restrict__ lengths, int bs,
                                                          int32_t* __restrict__ seq_starts,
                                                          int32_t* __restrict__ valid_cnt) {
  ptx::griddep_launch_dependents();
  ptx::griddep_wait();
  plan_scan_body(lengths, bs, seq_starts, valid_cnt);
}

// offsets[seq_starts[b] + j] = b*mx + j for j < len[b]  (the flat indices of
// the ones of a prefix-shaped mask, i.e. flatnonzero, packing.py:115).
// One CTA-slice per sequence, grid-strided.
__global__ void plan_offsets_kernel(const int32_t* __restrict__ seq_starts, int bs, int mx,
                                    int32_t* __restrict__ offsets) {
  ptx::griddep_launch_dependents();
  ptx::griddep_wait();
  for (int b = blockIdx.x; b < bs; b += gridDim.x) {
    const int s0 = seq_starts[b];
    const int len = seq_starts[b + 1] - s0;
    for (int j = threadIdx.x; j < len; j += blockDim.x) offsets[s0 + j] = b * mx + j;
  }
}

// ------------------------------------------------------------------ pack
__device__ __forceinline__ void load8(const float* p, float (&v)[8]) {
  const float4 a = __ldg(reinterpret_cast<const float4*>(p));
  const float4 b = __ldg(reinterpret_cast<const float4*>(p) + 1);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ void load8(const __nv_bfloat16* p, float (&v)[8]) {
  const uint4 a = __ldg(reinterpret_cast<const uint4*>(p));
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&a);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __bfloat1622float2(h[i]);
    v[2 * i] = f.x;
    v[2 * i + 1] = f.y;
  }
}
__device__ __forceinline__ void store8(float* p, const float (&v)[8]) {
  reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
  reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
}
__device__ __forceinline__ void store8(__nv_bfloat16* p, const float (&v)[8]) {
  uint4 o;
  o.x = ptx::pack_bf16x2(v[0], v[1]);
  o.y = ptx::pack_bf16x2(v[2], v[3]);
  o.z = ptx::pack_bf16x2(v[4], v[5]);
  o.w = ptx::pack_bf16x2(v[6], v[7]);
  *reinterpret_cast<uint4*>(p) = o;
}
__device__ __forceinline__ void zero8(float* p) {
  reinterpret_cast<float4*>(p)[0] = make_float4(0.f, 0.f, 0.f, 0.f);
  reinterpret_cast<float4*>(p)[1] = make_float4(0.f, 0.f, 0.f, 0.f);
}
__device__ __forceinline__ void zero8(__nv_bfloat16* p) { *reinterpret_cast<uint4*>(p) = make_uint4(0, 0, 0, 0); }

// Exact fp32 copies (pack/unpack in fp32 are bit copies, packing.py:148,159).
__device__ __forceinline__ void copy8(const float* s, float* d) {
  reinterpret_cast<float4*>(d)[0] = __ldg(reinterpret_cast<const float4*>(s));
  reinterpret_cast<float4*>(d)[1] = __ldg(reinterpret_cast<const float4*>(s) + 1);
}
__device__ __forceinline__ void copy8(const __nv_bfloat16* s, __nv_bfloat16* d) {
  *reinterpret_cast<uint4*>(d) = __ldg(reinterpret_cast<const uint4*>(s));
}
template <typename Tin, typename Tout>
__device__ __forceinline__ void move8(const Tin* s, Tout* d) {
  if constexpr (std::is_same<Tin, Tout>::value) {
    copy8(s, d);
  } else {
    float v[8];
    load8(s, v);
    store8(d, v);
  }
}

__device__ __forceinline__ float to_f(float v) { return v; }
__device__ __forceinline__ float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
template <typename T>
__device__ __forceinline__ T from_f(float v);
template <>
__device__ __forceinline__ float from_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

// Element-wise variants for widths that are not a multiple of 8 (the
// reference accepts any hidden width; the encoder itself uses k % 64 == 0).
template <typename Tin, typename Tout>
__global__ void pack_scalar_kernel(const Tin* __restrict__ padded, const int32_t* __restrict__ offsets, int T, int k,
                                   Tout* __restrict__ packed) {
  ptx::griddep_launch_dependents();
  ptx::griddep_wait();
  const long long total = static_cast<long long>(T) * k;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int row = static_cast<int>(i / k);
    const int c = static_cast<int>(i - static_cast<long long>(row) * k);
    packed[i] = from_f<Tout>(to_f(padded[static_cast<long long>(__ldg(offsets + row)) * k + c]));
  }
}
template <typename Tin, typename Tout>
__global__ void unpack_scalar_kernel(const Tin* __restrict__ packed, const int32_t* __restrict__ seq_starts, int bs,
                                     int mx, int k, Tout* __restrict__ padded) {
  ptx::griddep_launch_dependents();
  ptx::griddep_wait();
  const long long total = static_cast<long long>(bs) * mx * k;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long prow = i / k;
    const int c = static_cast<int>(i - prow * k);
    const int b = static_cast<int>(prow / mx);
    const int j = static_cast<int>(prow - static_cast<long long>(b) * mx);
    const int s0 = __ldg(seq_starts + b);
    const int len = __ldg(seq_starts + b + 1) - s0;
    padded[i] = j < len ? from_f<Tout>(to_f(packed[static_cast<long long>(s0 + j) * k + c])) : from_f<Tout>(0.f);
  }
}

template <typename Tin, typename Tout>
__global__ void pack_kernel(const Tin* __restrict__ padded, const int32_t* __restrict__ offsets, int T, int k,
                            Tout* __restrict__ packed) {
  ptx::griddep_launch_dependents();
  ptx::griddep_wait();
  const int chunks = k / 8;
  const long long total = static_cast<long long>(T) * chunks;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int row = static_cast<int>(i / chunks);
    const int c = static_cast<int>(i - static_cast<long long>(row) * chunks) * 8;
    const long long src = static_cast<long long>(__ldg(offsets + row)) * k + c;
    move8(padded + src, packed + static_cast<long long>(row) * k + c);
  }
}

// One pass over every padded row: valid rows copy from their packed row,
// padded rows are written with zeros (so no separate memset pass).
template <typename Tin, typename Tout>
__global__ void unpack_kernel(const Tin* __restrict__ packed, const int32_t* __restrict__ seq_starts, int bs,
                              int mx, int k, Tout* __restrict__ padded) {
  ptx::griddep_launch_dependents();
  ptx::griddep_wait();
  const int chunks = k / 8;
  const long long total = static_cast<long long>(bs) * mx * chunks;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long prow = i / chunks;
    const int c = static_cast<int>(i - prow * chunks) * 8;
    const int b = static_cast<int>(prow / mx);
    const int j = static_cast<int>(prow - static_cast<long long>(b) * mx);
    const int s0 = __ldg(seq_starts + b);
    const int len = __ldg(seq_starts + b + 1) - s0;
    Tout* dst = padded + prow * k + c;
    if (j < len) {
      move8(packed + static_cast<long long>(s0 + j) * k + c, dst);
    } else {
      zero8(dst);
    }
  }
}

static int grid_for(long long work_items, int threads) {
  const int sms = num_sms() > 0 ? num_sms() : 148;
  long long blocks = (work_items + threads - 1) / threads;
  const long long cap = static_cast<long long>(sms) * 8;  // 8 x 256-thread CTAs per SM resident
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  return static_cast<int>(blocks);
}

template <typename Tin, typename Tout>
static int launch_pack(const void* in, const int32_t* offsets, int T, int k, void* out, cudaStream_t s) {
  const int threads = 256;
  if (k % 8 == 0) {
    BT_LAUNCH((pack_kernel<Tin, Tout>), dim3(grid_for(static_cast<long long>(T) * (k / 8), threads)), dim3(threads), 0,
              s, 1, static_cast<const Tin*>(in), offsets, T, k, static_cast<Tout*>(out));
  } else {
    BT_LAUNCH((pack_scalar_kernel<Tin, Tout>), dim3(grid_for(static_cast<long long>(T) * k, threads)), dim3(threads), 0,
              s, 1, static_cast<const Tin*>(in), offsets, T, k, static_cast<Tout*>(out));
  }
  return BT_OK;
}
template <typename Tin, typename Tout>
static int launch_unpack(const void* in, const int32_t* starts, int bs, int mx, int k, void* out, cudaStream_t s) {
  const int threads = 256;
  if (k % 8 == 0) {
    BT_LAUNCH((unpack_kernel<Tin, Tout>), dim3(grid_for(static_cast<long long>(bs) * mx * (k / 8), threads)),
              dim3(threads), 0, s, 1, static_cast<const Tin*>(in), starts, bs, mx, k, static_cast<Tout*>(out));
  } else {
    BT_LAUNCH((unpack_scalar_kernel<Tin, Tout>), dim3(grid_for(static_cast<long long>(bs) * mx * k, threads)),
              dim3(threads), 0, s, 1, static_cast<const Tin*>(in), starts, bs, mx, k, static_cast<Tout*>(out));
  }
  return BT_OK;
}

}  // namespace bt

using namespace bt;

namespace bt {
// MHA work schedule: the sequences as (start row, length) sorted by
// descending 128-key block count (a counting sort; ties in any order -- the
// order only decides which CTAs the hardware dispatches first, never a
// result).  The MHA reads one int2 per CTA from it, so the longest attention
// problems start in the first wave and the short ones fill the tail (LPT),
// at no extra load latency per CTA.  One CTA.
constexpr int SCHED_MAX_BUCKETS = 1024;
__device__ __forceinline__ void plan_sched_body(const int32_t* __restrict__ seq_starts, int bs, int nbk,
                                                int2* __restrict__ sched, int* __restrict__ nunits,
                                                int2* __restrict__ units, int* __restrict__ nsegs,
                                                int4* __restrict__ segs) {
  // counting sort by key-block count (bucket 0 = the most blocks); a
  // sequence of nb blocks has nb query tiles, so a bucket's tile units are
  // contiguous: unit_base[bucket] + rank * nb
  __shared__ int cnt[SCHED_MAX_BUCKETS];
  __shared__ int ubase[SCHED_MAX_BUCKETS];
  __shared__ int bstart[SCHED_MAX_BUCKETS];
  for (int i = threadIdx.x; i < nbk; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < bs; i += blockDim.x) {
    const int len = seq_starts[i + 1] - seq_starts[i];
    atomicAdd(&cnt[min(nbk - 1, max(0, nbk - (len + 127) / 128))], 1);  // longest -> bucket 0
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0, urun = 0;
    for (int i = 0; i < nbk; ++i) {
      const int c = cnt[i];
      cnt[i] = run;
      bstart[i] = run;
      ubase[i] = urun;
      run += c;
      urun += c * (nbk - i);
    }
    nunits[0] = urun;
    nunits[1] = 0;  // the MHA tile-list queue: next item, finished CTAs
    nunits[2] = 0;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < bs; i += blockDim.x) {
    const int st = seq_starts[i], len = seq_starts[i + 1] - st;
    const int bk = min(nbk - 1, max(0, nbk - (len + 127) / 128));
    const int pos = atomicAdd(&cnt[bk], 1);
    sched[pos] = make_int2(st, len);
    const int nb = nbk - bk;
    int2* u = units + ubase[bk] + (pos - bstart[bk]) * nb;
    for (int q = 0; q < nb; ++q) u[q] = make_int2(st, (q << 20) | len);
  }
  // MHA segments (short batches): the query tiles of sequences longer than
  // 128 rows, then groups of adjacent sequences of <= 128 rows whose rows
  // fit one 128-row tile together (one key block; each row masked to its own
  // sequence), greedily from the left of each run of short sequences.  In
  // parallel over the sequences (a serial walk by one thread cost ~3 us at
  // bs = 16): each short sequence i finds where a group starting at i would
  // end (gend), each run start walks its chain of group starts, and two warp
  // scans place the long tiles and the groups -- the same list, in the same
  // order, as the serial greedy.
  if (segs != nullptr) {
    __shared__ int ss[SEG_MAX_BS + 1];
    __shared__ int gend[SEG_MAX_BS];
    __shared__ int ntile[SEG_MAX_BS];   // long: its query tiles; then exclusive offsets
    __shared__ int gstart[SEG_MAX_BS];  // 1 if a group starts at i; then exclusive offsets
    __shared__ int tot[2];
    for (int i = threadIdx.x; i <= bs; i += blockDim.x) ss[i] = seq_starts[i];
    __syncthreads();
    for (int i = threadIdx.x; i < bs; i += blockDim.x) {
      const int len = ss[i + 1] - ss[i];
      ntile[i] = len > 128 ? (len + 127) / 128 : 0;
      gstart[i] = 0;
      int j = i;
      if (len <= 128)
        while (j < bs && ss[j + 1] - ss[j] <= 128 && ss[j + 1] - ss[i] <= 128) ++j;
      gend[i] = j;  // the group [i, j) if one starts at i
    }
    __syncthreads();
    for (int i = threadIdx.x; i < bs; i += blockDim.x) {
      const bool shortseq = ss[i + 1] - ss[i] <= 128;
      if (shortseq && (i == 0 || ss[i] - ss[i - 1] > 128))
        for (int j = i; j < bs && ss[j + 1] - ss[j] <= 128; j = gend[j]) gstart[j] = 1;
    }
    __syncthreads();
    if (threadIdx.x < 64) {  // warp 0 scans ntile, warp 1 gstart (<= 8 entries per lane)
      int* a = threadIdx.x < 32 ? ntile : gstart;
      const int lane = threadIdx.x & 31, per = (bs + 31) / 32, b0 = min(bs, lane * per), b1 = min(bs, b0 + per);
      int run = 0;
      for (int i = b0; i < b1; ++i) run += a[i];
      int x = run;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      int off = x - run;
      for (int i = b0; i < b1; ++i) {
        const int v = a[i];
        a[i] = off;
        off += v;
      }
      if (lane == 31) tot[threadIdx.x >> 5] = x;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < bs; i += blockDim.x) {
      const int st = ss[i], en = ss[i + 1];
      if (en - st > 128) {
        int n = ntile[i];
        for (int q = st; q < en; q += 128, ++n) {
          segs[2 * n] = make_int4(st, en, q, min(en, q + 128));
          segs[2 * n + 1] = make_int4(i, i, 0, 0);
        }
      } else {
        const bool starts = (i + 1 < bs ? gstart[i + 1] : tot[1]) != gstart[i];
        if (starts) {
          const int n = tot[0] + gstart[i], e = gend[i];
          segs[2 * n] = make_int4(st, ss[e], st, ss[e]);
          segs[2 * n + 1] = make_int4(i, e - 1, 0, 0);
        }
      }
    }
    if (threadIdx.x == 0) *nsegs = tot[0] + tot[1];
  }
}

__global__ void __launch_bounds__(1024) plan_sched_kernel(const int32_t* __restrict__ seq_starts, int bs, int nbk,
                                                           int2* __restrict__ sched, int* __restrict__ nunits,
                                                           int2* __restrict__ units, int* __restrict__ nsegs,
                                                           int4* __restrict__ segs) {
  ptx::griddep_launch_dependents();
  ptx::griddep_wait();
  plan_sched_body(seq_starts, bs, nbk, sched, nunits, units, nsegs, segs);
}

constexpr int PLAN_SMEM_BS = 4096;
// The forward's whole plan in one CTA: lengths -> seq_starts, then the MHA
// schedule (what plan_scan_kernel + plan_sched_kernel do in two launches).
__global__ void __launch_bounds__(1024) plan_forward_kernel(const int32_t* __restrict__ lengths, int bs, int nbk,
                                                             int32_t* __restrict__ seq_starts,
                                                             int2* __restrict__ sched, int* __restrict__ nunits,
                                                             int2* __restrict__ units, int* __restrict__ nsegs,
                                                             int4* __restrict__ segs) {
  // seq_starts also kept in shared memory (bs <= PLAN_SMEM_BS) so the
  // schedule reads no global memory
  __shared__ int32_t sm_starts[PLAN_SMEM_BS + 1];
  ptx::griddep_launch_dependents();
  ptx::griddep_wait();
  const bool in_smem = bs <= PLAN_SMEM_BS;
  plan_scan_body(lengths, bs, seq_starts, nullptr, in_smem ? sm_starts : nullptr);
  __syncthreads();  // seq_starts written by this CTA is visible to all its threads
  plan_sched_body(in_smem ? sm_starts : seq_starts, bs, nbk, sched, nunits, units, nsegs, segs);
}

// Pack by sequence starts (no offsets array): padded row b*mx + j -> packed
// row seq_starts[b] + j for j < len[b]; padded rows are skipped.
template <typename Tin, typename Tout>
__global__ void pack_starts_kernel(const Tin* __restrict__ padded, const int32_t* __restrict__ seq_starts, int bs,
                                   int mx, int k, Tout* __restrict__ packed) {
  ptx::griddep_launch_dependents();
  ptx::griddep_wait();
  const int chunks = k / 8;
  const long long total = static_cast<long long>(bs) * mx * chunks;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long prow = i / chunks;
    const int c = static_cast<int>(i - prow * chunks) * 8;
    const int b = static_cast<int>(prow / mx);
    const int j = static_cast<int>(prow - static_cast<long long>(b) * mx);
    const int s0 = __ldg(seq_starts + b);
    if (j < __ldg(seq_starts + b + 1) - s0) move8(padded + prow * k + c, packed + static_cast<long long>(s0 + j) * k + c);
  }
}

// ---------------------------------------------------------------- forward prologue
// The whole front of the forward in ONE launch (what plan_forward + pack_starts
// do in two, plus the zeroing half of unpack): every CTA scans the lengths into
// shared memory; CTA 0 publishes seq_starts and writes the MHA schedule
// (plan_sched_body) while the other CTAs, one warp per row, gather the valid
// rows fp32 -> bf16 (packed row r -> sequence b by a binary search over the
// starts), record where each packed row goes in the padded output (row_map,
// read by the last layer's LayerNorm, which writes the output rows itself),
// and zero the output's padded rows (packing.py:158-159: exact zeros).
// PADDED = false: the input is already packed ([T, k] fp32, e2e host path).
constexpr int PRO_THREADS = 512;
constexpr int PRO_MAX_BS = 4096;

// Exclusive scan of lengths[0..bs) into ss[0..bs] (shared memory), any block
// size that is a multiple of 32.
__device__ __forceinline__ void block_scan_lengths(const int32_t* __restrict__ lengths, int bs, int32_t* ss) {
  __shared__ int32_t wsum[32];
  __shared__ int32_t carry_s;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  if (tid == 0) carry_s = 0;
  __syncthreads();
  for (int base = 0; base < bs; base += blockDim.x) {
    const int i = base + tid;
    const int v = (i < bs) ? __ldg(lengths + i) : 0;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[wid] = x;
    __syncthreads();
    if (wid == 0) {
      int w = lane < nw ? wsum[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      wsum[lane] = w;
    }
    __syncthreads();
    const int incl = x + (wid ? wsum[wid - 1] : 0) + carry_s;
    if (i < bs) ss[i] = incl - v;
    __syncthreads();
    if (tid == blockDim.x - 1) carry_s = incl;
    __syncthreads();
  }
  if (tid == 0) ss[bs] = carry_s;
  __syncthreads();
}

template <bool PADDED>
__global__ void __launch_bounds__(PRO_THREADS) forward_prologue_kernel(
    const int32_t* __restrict__ lengths, int bs, int mx, int nbk, int k, const float* __restrict__ x_in,
    __nv_bfloat16* __restrict__ x_out, int32_t* __restrict__ seq_starts, int2* __restrict__ sched,
    int* __restrict__ nunits, int2* __restrict__ units, int* __restrict__ nsegs, int4* __restrict__ segs,
    float* __restrict__ out_padded, int32_t* __restrict__ row_map) {
  __shared__ int32_t ss[PRO_MAX_BS + 1];
  ptx::griddep_launch_dependents();
  ptx::griddep_wait();  // lengths / input / output may belong to earlier work on the stream
  block_scan_lengths(lengths, bs, ss);
  if (blockIdx.x == 0) {
    for (int i = threadIdx.x; i <= bs; i += blockDim.x) seq_starts[i] = ss[i];
    plan_sched_body(ss, bs, nbk, sched, nunits, units, nsegs, segs);
    return;
  }
  const int T = ss[bs];
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  const int nwarps = (gridDim.x - 1) * wpb;
  const int gw = (blockIdx.x - 1) * wpb + (threadIdx.x >> 5);
  const int nchunk = k >> 3;
  for (int r = gw; r < T; r += nwarps) {
    long long src = r;
    if (PADDED) {
      int lo = 0, hi = bs - 1;  // sequence of packed row r: the last b with ss[b] <= r
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (ss[mid] <= r) lo = mid; else hi = mid - 1;
      }
      src = static_cast<long long>(lo) * mx + (r - ss[lo]);
      if (lane == 0) row_map[r] = static_cast<int32_t>(src);
    }
    const float* srow = x_in + src * k;
    __nv_bfloat16* drow = x_out + static_cast<long long>(r) * k;
    if (nchunk <= 128) {
      // every load of the row in flight before any use (k <= 1024: <= 4 chunks per lane)
      float4 v[4][2];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int c = lane + 32 * i;
        if (c < nchunk) {
          v[i][0] = __ldg(reinterpret_cast<const float4*>(srow) + 2 * c);
          v[i][1] = __ldg(reinterpret_cast<const float4*>(srow) + 2 * c + 1);
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int c = lane + 32 * i;
        if (c < nchunk)
          reinterpret_cast<uint4*>(drow)[c] =
              make_uint4(ptx::pack_bf16x2(v[i][0].x, v[i][0].y), ptx::pack_bf16x2(v[i][0].z, v[i][0].w),
                         ptx::pack_bf16x2(v[i][1].x, v[i][1].y), ptx::pack_bf16x2(v[i][1].z, v[i][1].w));
      }
    } else {
      for (int c = lane; c < nchunk; c += 32) move8(srow + c * 8, drow + c * 8);
    }
  }
  if (PADDED) {
    // padded row q (0 <= q < bs*mx - T) is in sequence b = the last b whose
    // preceding sequences hold <= q padded rows (b*mx - ss[b] of them)
    const int nz = bs * mx - T;
    const int k4 = k >> 2;
    for (int q = gw; q < nz; q += nwarps) {
      int lo = 0, hi = bs - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (mid * mx - ss[mid] <= q) lo = mid; else hi = mid - 1;
      }
      const long long prow = static_cast<long long>(lo) * mx + (ss[lo + 1] - ss[lo]) + (q - (lo * mx - ss[lo]));
      float4* o = reinterpret_cast<float4*>(out_padded + prow * k);
      for (int c = lane; c < k4; c += 32) o[c] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
}

}  // namespace bt

extern "C" {

int bt_version(void) { return 1; }
const char* bt_last_error(void) { return bt::last_error(); }
long long bt_launch_count(void) { return bt::g_launches.load(); }
int bt_num_sms(void) { return bt::num_sms(); }

int bt_plan_mask(const uint8_t* mask, int bs, int mx, int32_t* lengths, int32_t* seq_starts, int32_t* offsets,
                 int32_t* valid_cnt_dev, int32_t* status_dev, bt_stream_t stream) {
  BT_REQUIRE(bs >= 1 && mx >= 1, BT_ESHAPE, "mask must be at least 1x1, got %dx%d", bs, mx);
  BT_REQUIRE(static_cast<long long>(bs) * mx < (1LL << 31), BT_ESHAPE, "mask too large (%d x %d)", bs, mx);
  BT_REQUIRE(mask && lengths && seq_starts && offsets && status_dev, BT_ESHAPE, "null pointer");
  cudaStream_t s = as_stream(stream);
  BT_CUDA_CHECK(cudaMemsetAsync(status_dev, 0, sizeof(int32_t), s));
  const int warps = 8;
  const int sms = num_sms() > 0 ? num_sms() : 148;
  int grid = (bs + warps - 1) / warps;
  if (grid > sms * 8) grid = sms * 8;
  BT_LAUNCH(plan_rows_kernel, dim3(grid), dim3(warps * 32), 0, s, 1, mask, bs, mx, lengths, status_dev);
  BT_LAUNCH(plan_scan_kernel, dim3(1), dim3(1024), 0, s, 1, (const int32_t*)lengths, bs, seq_starts, valid_cnt_dev);
  BT_LAUNCH(plan_offsets_kernel, dim3(bs < sms * 4 ? bs : sms * 4), dim3(256), 0, s, 1, (const int32_t*)seq_starts,
            bs, mx, offsets);
  return BT_OK;
}

int bt_plan_lengths(const int32_t* lengths, int bs, int mx, int32_t* seq_starts, int32_t* offsets,
                    bt_stream_t stream) {
  BT_REQUIRE(bs >= 1 && mx >= 1, BT_ESHAPE, "batch must be at least 1x1, got %dx%d", bs, mx);
  BT_REQUIRE(lengths && seq_starts, BT_ESHAPE, "null pointer");
  cudaStream_t s = as_stream(stream);
  const int sms = num_sms() > 0 ? num_sms() : 148;
  BT_LAUNCH(plan_scan_kernel, dim3(1), dim3(1024), 0, s, 1, lengths, bs, seq_starts, (int32_t*)nullptr);
  if (offsets) {
    BT_LAUNCH(plan_offsets_kernel, dim3(bs < sms * 4 ? bs : sms * 4), dim3(256), 0, s, 1, (const int32_t*)seq_starts,
              bs, mx, offsets);
  }
  return BT_OK;
}

int bt_plan_sched(const int32_t* seq_starts, int bs, int mx, void* sched, bt_stream_t stream) {
  BT_REQUIRE(bs >= 1 && mx >= 1 && seq_starts && sched, BT_ESHAPE, "plan_sched: bad arguments");
  const int nbk = (mx + 127) / 128;
  BT_REQUIRE(nbk <= SCHED_MAX_BUCKETS, BT_ESHAPE, "plan_sched: max_seq_len %d too large", mx);
  BT_REQUIRE((mx + 127) / 128 < 2048 && mx < (1 << 20), BT_ESHAPE, "plan_sched: max_seq_len %d too large", mx);
  uint8_t* base = static_cast<uint8_t*>(sched);
  int* nunits = reinterpret_cast<int*>(base + sched_units_offset(bs));
  BT_LAUNCH(plan_sched_kernel, dim3(1), dim3(1024), 0, as_stream(stream), 1, seq_starts, bs, nbk,
            static_cast<int2*>(sched), nunits, reinterpret_cast<int2*>(nunits + 4),
            reinterpret_cast<int*>(base + sched_segs_offset(bs, mx)),
            bs <= SEG_MAX_BS && mx <= SEG_MAX_MX ? reinterpret_cast<int4*>(base + sched_segs_offset(bs, mx) + 16)
                                                 : nullptr);
  return BT_OK;
}

// The forward's plan (bt_encoder_forward): seq_starts + MHA schedule in one
// launch, and the pack from seq_starts (no offsets array).
int bt_plan_forward(const int32_t* lengths, int bs, int mx, int32_t* seq_starts, void* sched,
                             bt_stream_t stream) {
  BT_REQUIRE(bs >= 1 && mx >= 1 && lengths && seq_starts && sched, BT_ESHAPE, "plan_forward: bad arguments");
  const int nbk = (mx + 127) / 128;
  BT_REQUIRE(nbk <= SCHED_MAX_BUCKETS && mx < (1 << 20), BT_ESHAPE, "plan_forward: max_seq_len %d too large", mx);
  uint8_t* base = static_cast<uint8_t*>(sched);
  int* nunits = reinterpret_cast<int*>(base + sched_units_offset(bs));
  BT_LAUNCH(plan_forward_kernel, dim3(1), dim3(1024), 0, as_stream(stream), 1, lengths, bs, nbk, seq_starts,
            static_cast<int2*>(sched), nunits, reinterpret_cast<int2*>(nunits + 4),
            reinterpret_cast<int*>(base + sched_segs_offset(bs, mx)),
            bs <= SEG_MAX_BS && mx <= SEG_MAX_MX ? reinterpret_cast<int4*>(base + sched_segs_offset(bs, mx) + 16)
                                                 : nullptr);
  return BT_OK;
}

int bt_pack_starts(const float* padded, const int32_t* seq_starts, int bs, int mx, int k, void* packed_bf16,
                            bt_stream_t stream) {
  BT_REQUIRE(bs >= 1 && mx >= 1 && k >= 8 && k % 8 == 0, BT_ESHAPE, "pack_starts: bad shape");
  const int threads = 256;
  BT_LAUNCH((pack_starts_kernel<float, __nv_bfloat16>), dim3(grid_for(static_cast<long long>(bs) * mx * (k / 8), threads)),
            dim3(threads), 0, as_stream(stream), 1, padded, seq_starts, bs, mx, k,
            static_cast<__nv_bfloat16*>(packed_bf16));
  return BT_OK;
}

// The forward's front in one launch (forward_prologue_kernel).  x_padded
// non-null: padded fp32 input [bs*mx, k], its packed bf16 rows go to x_packed,
// row_map[T] receives each packed row's padded row and out_padded's padded
// rows are zeroed; x_padded null: x_packed_in [T, k] fp32 is converted.
int bt_forward_prologue(const int32_t* lengths, int bs, int mx, int k, const float* x_padded,
                        const float* x_packed_in, void* x_packed, int32_t* seq_starts, void* sched, float* out_padded,
                        int32_t* row_map, int T, bt_stream_t stream) {
  BT_REQUIRE(lengths && x_packed && seq_starts && sched && (x_padded ? out_padded && row_map : x_packed_in != nullptr),
             BT_ESHAPE, "forward_prologue: null pointer");
  BT_REQUIRE(bs >= 1 && bs <= PRO_MAX_BS && mx >= 1 && k >= 8 && k % 8 == 0 && T >= 1, BT_ESHAPE,
             "forward_prologue: bad shape bs=%d mx=%d k=%d", bs, mx, k);
  const int nbk = (mx + 127) / 128;
  BT_REQUIRE(nbk <= SCHED_MAX_BUCKETS && mx < (1 << 20), BT_ESHAPE, "forward_prologue: max_seq_len %d too large", mx);
  uint8_t* base = static_cast<uint8_t*>(sched);
  int* nunits = reinterpret_cast<int*>(base + sched_units_offset(bs));
  int4* segs = bs <= SEG_MAX_BS && mx <= SEG_MAX_MX ? reinterpret_cast<int4*>(base + sched_segs_offset(bs, mx) + 16)
                                                    : nullptr;
  int* nsegs = reinterpret_cast<int*>(base + sched_segs_offset(bs, mx));
  const int sms = num_sms() > 0 ? num_sms() : 148;
  const long long rows = x_padded ? std::max<long long>(T, static_cast<long long>(bs) * mx - T) : T;
  const int wpb = PRO_THREADS / 32;
  const int grid = 1 + static_cast<int>(std::min<long long>(sms * 4LL, (rows + wpb - 1) / wpb));
  if (x_padded) {
    BT_LAUNCH(forward_prologue_kernel<true>, dim3(grid), dim3(PRO_THREADS), 0, as_stream(stream), 1, lengths, bs, mx,
              nbk, k, x_padded, static_cast<__nv_bfloat16*>(x_packed), seq_starts, static_cast<int2*>(sched), nunits,
              reinterpret_cast<int2*>(nunits + 4), nsegs, segs, out_padded, row_map);
  } else {
    BT_LAUNCH(forward_prologue_kernel<false>, dim3(grid), dim3(PRO_THREADS), 0, as_stream(stream), 1, lengths, bs,
              mx, nbk, k, x_packed_in, static_cast<__nv_bfloat16*>(x_packed), seq_starts, static_cast<int2*>(sched),
              nunits, reinterpret_cast<int2*>(nunits + 4), nsegs, segs, static_cast<float*>(nullptr),
              static_cast<int32_t*>(nullptr));
  }
  return BT_OK;
}

size_t bt_plan_sched_bytes(int bs, int mx) { return bs >= 1 && mx >= 1 ? sched_bytes(bs, mx) : 0; }

int bt_pack(const void* padded, int in_dtype, const int32_t* offsets, int T, int k, void* packed, int out_dtype,
            bt_stream_t stream) {
  BT_REQUIRE(T >= 0 && k >= 1, BT_ESHAPE, "pack: need T >= 0 and k >= 1, got T=%d k=%d", T, k);
  BT_REQUIRE((in_dtype == BT_F32 || in_dtype == BT_BF16) && (out_dtype == BT_F32 || out_dtype == BT_BF16), BT_ECONFIG,
             "pack: unsupported dtypes %d -> %d", in_dtype, out_dtype);
  if (T == 0) return BT_OK;
  cudaStream_t s = as_stream(stream);
  if (in_dtype == BT_F32 && out_dtype == BT_BF16) return launch_pack<float, __nv_bfloat16>(padded, offsets, T, k, packed, s);
  if (in_dtype == BT_F32) return launch_pack<float, float>(padded, offsets, T, k, packed, s);
  if (out_dtype == BT_BF16) return launch_pack<__nv_bfloat16, __nv_bfloat16>(padded, offsets, T, k, packed, s);
  return launch_pack<__nv_bfloat16, float>(padded, offsets, T, k, packed, s);
}

int bt_unpack(const void* packed, int in_dtype, const int32_t* seq_starts, int bs, int mx, int k, void* padded,
              int out_dtype, bt_stream_t stream) {
  BT_REQUIRE(bs >= 1 && mx >= 1 && k >= 1, BT_ESHAPE, "unpack: bad shape bs=%d mx=%d k=%d", bs, mx, k);
  BT_REQUIRE((in_dtype == BT_F32 || in_dtype == BT_BF16) && (out_dtype == BT_F32 || out_dtype == BT_BF16), BT_ECONFIG,
             "unpack: unsupported dtypes %d -> %d", in_dtype, out_dtype);
  cudaStream_t s = as_stream(stream);
  if (in_dtype == BT_BF16 && out_dtype == BT_F32) return launch_unpack<__nv_bfloat16, float>(packed, seq_starts, bs, mx, k, padded, s);
  if (in_dtype == BT_F32 && out_dtype == BT_F32) return launch_unpack<float, float>(packed, seq_starts, bs, mx, k, padded, s);
  if (in_dtype == BT_BF16) return launch_unpack<__nv_bfloat16, __nv_bfloat16>(packed, seq_starts, bs, mx, k, padded, s);
  return launch_unpack<float, __nv_bfloat16>(packed, seq_starts, bs, mx, k, padded, s);
}

}  // extern "C"
