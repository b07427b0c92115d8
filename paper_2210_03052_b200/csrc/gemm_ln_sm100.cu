// Fused projection GEMM + add-bias + residual + LayerNorm (reference
// encoder.py:385-388 and :404-407: proj = x W; y = LN((proj + residual) +
// bias), fusion.py:79-98; paper section III-C1 fuses the same three steps
// after GEMM #1 / #3):
//
//   Y[M, N] = LN( (A[M,K] * Bt[N,K]^T + R[M,N]) + bias ) * gamma + beta
//
// A LayerNorm row needs all N columns, but a 128 x N fp32 tile (N = 768 /
// 1024) does not fit one SM's TMEM next to a pipeline.  So one row block is
// computed by a CLUSTER of CL = N / 128 CTAs, each owning a 128 x 128 tile
// (tcgen05.mma cta_group::1, fp32 accumulator in 128 TMEM columns):
//
//   warp 0      TMA producer: A / B k-blocks -> 4-stage 128B-swizzled ring;
//               the residual tile (128 x 128 bf16) once, on its own barrier
//   warp 1      TMEM allocator + single-thread MMA issuer (elect.sync)
//   warps 2-9   epilogue, two threads per row (warp w: TMEM lanes 32*(w%4),
//               columns 64*((w-2)/4) .. +63): v = (acc + residual) + bias in
//               64 registers; each thread's (mean, M2) over its 64 columns
//               goes to every CTA of the cluster through DSMEM
//               (st.shared::cluster), one cluster barrier, then the 2*CL
//               partials of a row are combined with the parallel-variance
//               formula (mean = avg of means, M2 = sum M2_i + n sum (mean_i -
//               mean)^2 -- exact, no one-pass E[x^2] - E[x]^2), normalised and
//               written as bf16 through shared memory with TMA stores.
//               bias / gamma / beta are staged in shared memory while the
//               mainloop runs.
//
// The proj tensor never reaches memory and the separate LayerNorm launch
// (and its re-read of proj and residual) disappears.  Used when the row
// blocks fit one wave of clusters (cudaOccupancyMaxActiveClusters); otherwise
// the encoder keeps GEMM + ln_bias_residual_kernel.

#include "common.cuh"
#include "ptx.cuh"
#include "tma_host.cuh"

namespace bt {

// GLN_MCAST = 1: the CL CTAs of a cluster share one row block of A, so each
// A k-block is TMA-loaded ONCE per cluster (by CTA kb % CL) and multicast
// into every CTA's ring; a ring stage is refilled only after all CL MMA
// issuers have released it (their commits multicast to every CTA's empty
// barrier).  L2 -> SM traffic per cluster drops from CL x (A + B) to
// A + CL x B per k-block.  Correct (the GEMM+LN tests pass with it) but
// measured SLOWER at C2: 8.8 vs 8.3 us per launch (the cluster-wide stage
// release puts the six CTAs in lockstep; the per-SM feed is not what the L2
// dedup of the six simultaneous unicast loads leaves short).  0 (default):
// every CTA loads its own copy of A.
#ifndef GLN_MCAST
#define GLN_MCAST 0
#endif

constexpr int GLN_BN = 128;
constexpr int GLN_BK = 64;
constexpr int GLN_STAGES = 5;
constexpr int GLN_THREADS = 320;  // warp 0 TMA, warp 1 MMA, warps 2-9 epilogue
constexpr uint32_t GLN_TILE = 128 * GLN_BK * 2;  // 16 KB: one 128 x 64 bf16 operand tile

struct GlnCfg {
  static constexpr uint32_t A_OFF = 0;
  static constexpr uint32_t B_OFF = A_OFF + GLN_STAGES * GLN_TILE;
  static constexpr uint32_t R_OFF = B_OFF + GLN_STAGES * GLN_TILE;  // residual in, Y out: 2 boxes of 128 x 64
  static constexpr uint32_t ST_OFF = R_OFF + 2 * GLN_TILE;           // [16][128] float2 (mean, M2) partials
  static constexpr uint32_t PRM_OFF = ST_OFF + 16 * 128 * 8;         // bias, gamma, beta: 3 x 128 fp32
  static constexpr uint32_t BAR_OFF = PRM_OFF + 3 * 128 * 4;
  static constexpr size_t SMEM = 1024 + BAR_OFF + 256;
};

struct GlnParams {
  int M, N, K, num_k;
  const float* bias;
  const float* gamma;
  const float* beta;
  float eps;
};

__device__ __forceinline__ void st_cluster_f2(uint32_t addr, float a, float b) {
  asm volatile("st.shared::cluster.v2.f32 [%0], {%1, %2};" ::"r"(addr), "f"(a), "f"(b) : "memory");
}

__device__ __forceinline__ void named_bar_sync_gln(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
// tie a register array to a preceding tcgen05.wait::ld
__device__ __forceinline__ void gln_reg_tie(uint32_t (&r)[32]) {
  asm volatile(""
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                 "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]),
                 "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]),
                 "+r"(r[29]), "+r"(r[30]), "+r"(r[31]));
}

// byte offset of 16 B chunk j (0..15 over 128 columns) of row r in the two
// 128B-swizzled 128 x 64 boxes
__device__ __forceinline__ uint32_t r_off(int r, int j) {
  return static_cast<uint32_t>((j >> 3) * GLN_TILE + r * 128 + (((j & 7) ^ (r & 7)) << 4));
}

template <int CL>
__global__ void __launch_bounds__(GLN_THREADS, 1)
    gemm_ln_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmR, const __grid_constant__ CUtensorMap tmY,
                   const GlnParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem + GlnCfg::A_OFF;
  uint8_t* sB = smem + GlnCfg::B_OFF;
  uint8_t* sR = smem + GlnCfg::R_OFF;
  float2* stats = reinterpret_cast<float2*>(smem + GlnCfg::ST_OFF);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + GlnCfg::BAR_OFF);
  uint64_t* empty = full + GLN_STAGES;
  uint64_t* tfull = empty + GLN_STAGES;
  uint64_t* rfull = tfull + 1;
  uint32_t* holder = reinterpret_cast<uint32_t*>(rfull + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = static_cast<int>(ptx::cluster_ctarank());
  const int rb = blockIdx.x / CL;
  const int n0 = rank * GLN_BN;
  const int row_base = rb * 128;

  constexpr uint16_t all_ctas = static_cast<uint16_t>((1u << CL) - 1u);
  if (threadIdx.x == 0) {
    for (int s = 0; s < GLN_STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], GLN_MCAST ? CL : 1);  // multicast A: every CTA's MMA must release the stage
    }
    ptx::mbar_init(tfull, 1);
    ptx::mbar_init(rfull, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) {
    ptx::tmem_alloc(holder, 128);
    ptx::tmem_relinquish();
  }
  ptx::tc_fence_before();
  if (GLN_MCAST) {
    ptx::cluster_sync();  // every CTA's barriers exist before any multicast load / commit reaches them
  } else {
    __syncthreads();
  }
  ptx::tc_fence_after();
  const uint32_t tmem = *holder;
  ptx::griddep_launch_dependents();

  if (warp == 0) {
    // ---------------- TMA producer (warp-uniform loop, one elected lane issues)
    if (ptx::elect_one()) {
      ptx::prefetch_tmap(&tmA);
      ptx::prefetch_tmap(&tmB);
      ptx::prefetch_tmap(&tmR);
      ptx::prefetch_tmap(&tmY);
    }
    // weights do not depend on the previous kernel: the first stages' B
    // loads go out before griddepcontrol.wait
    const int pre = min(GLN_STAGES, p.num_k);
    for (int i = 0; i < pre; ++i) {
      if (ptx::elect_one()) {
        ptx::mbar_arrive_expect_tx(&full[i], 2 * GLN_TILE);
        ptx::tma_load_2d(sB + i * GLN_TILE, &tmB, &full[i], i * GLN_BK, n0);
      }
      __syncwarp();
    }
    ptx::griddep_wait();  // A and the residual are produced by earlier kernels
    if (ptx::elect_one()) {
      ptx::mbar_arrive_expect_tx(rfull, 2 * GLN_TILE);
      ptx::tma_load_2d(sR, &tmR, rfull, n0, row_base);
      ptx::tma_load_2d(sR + GLN_TILE, &tmR, rfull, n0 + 64, row_base);
    }
    __syncwarp();
    for (int kb = 0; kb < p.num_k; ++kb) {
      const int stage = kb % GLN_STAGES;
      if (kb >= GLN_STAGES) ptx::mbar_wait(&empty[stage], ((kb / GLN_STAGES) - 1) & 1);
      if (ptx::elect_one()) {
        if (kb >= pre) {
          ptx::mbar_arrive_expect_tx(&full[stage], 2 * GLN_TILE);
          ptx::tma_load_2d(sB + stage * GLN_TILE, &tmB, &full[stage], kb * GLN_BK, n0);
        }
        if (GLN_MCAST) {
          if (kb % CL == rank)
            ptx::tma_load_2d_mc(sA + stage * GLN_TILE, &tmA, &full[stage], kb * GLN_BK, row_base, all_ctas);
        } else {
          ptx::tma_load_2d(sA + stage * GLN_TILE, &tmA, &full[stage], kb * GLN_BK, row_base);
        }
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer: 128 x 128 x 16 per instruction
    constexpr uint32_t idesc = ptx::idesc_bf16(128, GLN_BN, false, false);
    const uint32_t a_base = ptx::smem_u32(sA), b_base = ptx::smem_u32(sB);
    for (int kb = 0; kb < p.num_k; ++kb) {
      const int stage = kb % GLN_STAGES;
      ptx::mbar_wait(&full[stage], (kb / GLN_STAGES) & 1);
      ptx::tc_fence_after();
      const uint64_t ad = ptx::sdesc_sw128(a_base + stage * GLN_TILE, 1024, 16);
      const uint64_t bd = ptx::sdesc_sw128(b_base + stage * GLN_TILE, 1024, 16);
      if (ptx::elect_one()) {
#pragma unroll
        for (int k = 0; k < GLN_BK / 16; ++k) ptx::mma_bf16_ss(tmem, ad + 2 * k, bd + 2 * k, idesc, (kb | k) ? 1u : 0u);
        if (GLN_MCAST)
          ptx::mma_commit_mc(&empty[stage], all_ctas);
        else
          ptx::mma_commit(&empty[stage]);
      }
      __syncwarp();
    }
    if (ptx::elect_one()) ptx::mma_commit(tfull);
    __syncwarp();
  }

  // ---------------- epilogue part 1: v = (acc + residual) + bias, local row stats
  const int quarter = warp & 3;
  const int half = (warp - 2) >> 2;  // epilogue warps: column half 0 / 1
  const int row = quarter * 32 + lane;
  float* prm = reinterpret_cast<float*>(smem + GlnCfg::PRM_OFF);  // [0,128) bias, [128,256) gamma, [256,384) beta
  float v[64];
  if (warp >= 2) {
    {  // stage this CTA's 128 columns of the parameters (overlaps the mainloop)
      const int t = threadIdx.x - 64;  // 0..255
      if (t < 128) {
        prm[t] = __ldg(p.bias + n0 + t);
      } else {
        prm[128 + (t - 128)] = __ldg(p.gamma + n0 + (t - 128));
        prm[256 + (t - 128)] = __ldg(p.beta + n0 + (t - 128));
      }
      named_bar_sync_gln(1, 256);
    }
    ptx::mbar_wait(rfull, 0);
    ptx::mbar_wait(tfull, 0);
    ptx::tc_fence_after();
    const uint32_t tcol = tmem + (static_cast<uint32_t>(quarter * 32) << 16) + half * 64;
    uint32_t r0[32], r1[32];
    ptx::tmem_ld32(tcol, r0);
    ptx::tmem_ld32(tcol + 32, r1);
    ptx::tmem_wait_ld(r0);
    gln_reg_tie(r1);
#pragma unroll
    for (int q = 0; q < 8; ++q) {  // 8 columns per 16 B residual chunk
      const int c0 = half * 64 + 8 * q;  // column within the CTA's 128
      const uint4 rv = *reinterpret_cast<const uint4*>(sR + r_off(row, c0 >> 3));
      const __nv_bfloat162* rh = reinterpret_cast<const __nv_bfloat162*>(&rv);
      const float4 b0 = *reinterpret_cast<const float4*>(prm + c0);
      const float4 b1 = *reinterpret_cast<const float4*>(prm + c0 + 4);
      const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 rf = __bfloat1622float2(rh[e]);
        const int i = 8 * q + 2 * e;
        const uint32_t a0 = i < 32 ? r0[i] : r1[i - 32];
        const uint32_t a1 = i + 1 < 32 ? r0[i + 1] : r1[i + 1 - 32];
        v[i] = (__uint_as_float(a0) + rf.x) + bb[2 * e];  // (x + residual) + bias, fusion.py:96
        v[i + 1] = (__uint_as_float(a1) + rf.y) + bb[2 * e + 1];
      }
    }
    float s4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int i = 0; i < 64; ++i) s4[i & 3] += v[i];
    const float mean_l = ((s4[0] + s4[1]) + (s4[2] + s4[3])) * (1.0f / 64);
    float q4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int i = 0; i < 64; ++i) {
      const float d = v[i] - mean_l;
      q4[i & 3] = fmaf(d, d, q4[i & 3]);
    }
    const float m2_l = (q4[0] + q4[1]) + (q4[2] + q4[3]);
    const uint32_t mine = ptx::smem_u32(&stats[(2 * rank + half) * 128 + row]);
#pragma unroll
    for (int r = 0; r < CL; ++r) st_cluster_f2(ptx::mapa_shared(mine, r), mean_l, m2_l);
  }
  ptx::cluster_sync();  // every CTA's row partials have landed in every CTA

  if (warp >= 2) {
    // ---------------- epilogue part 2: combine the 2*CL partials (n = 64 each), normalise, store
    float mean = 0.f;
#pragma unroll
    for (int r = 0; r < 2 * CL; ++r) mean += stats[r * 128 + row].x;
    mean *= 1.0f / (2 * CL);
    float m2 = 0.f;
#pragma unroll
    for (int r = 0; r < 2 * CL; ++r) {
      const float2 st = stats[r * 128 + row];
      const float d = st.x - mean;
      m2 += st.y + 64.0f * d * d;
    }
    const float rstd = 1.0f / sqrtf(m2 * (1.0f / (GLN_BN * CL)) + p.eps);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int c0 = half * 64 + 8 * j;
      const float4 g0 = *reinterpret_cast<const float4*>(prm + 128 + c0);
      const float4 g1 = *reinterpret_cast<const float4*>(prm + 128 + c0 + 4);
      const float4 e0 = *reinterpret_cast<const float4*>(prm + 256 + c0);
      const float4 e1 = *reinterpret_cast<const float4*>(prm + 256 + c0 + 4);
      const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
      const float ee[8] = {e0.x, e0.y, e0.z, e0.w, e1.x, e1.y, e1.z, e1.w};
      uint32_t w[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int i = 8 * j + 2 * e;
        w[e] = ptx::pack_bf16x2(gg[2 * e] * ((v[i] - mean) * rstd) + ee[2 * e],
                                gg[2 * e + 1] * ((v[i + 1] - mean) * rstd) + ee[2 * e + 1]);
      }
      *reinterpret_cast<uint4*>(sR + r_off(row, c0 >> 3)) = make_uint4(w[0], w[1], w[2], w[3]);
    }
    ptx::fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0 && row_base + quarter * 32 < p.M) {
      // this warp's 32-row slab of its 64-column box
      ptx::tma_store_2d(&tmY, sR + half * GLN_TILE + quarter * 32 * 128, n0 + 64 * half, row_base + quarter * 32);
      ptx::bulk_commit_group();
      ptx::bulk_wait_group<0>();
    }
    __syncwarp();
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 128);
  }
}

template <int CL>
static int launch_gln(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tr, const CUtensorMap& ty,
                      const GlnParams& p, cudaStream_t s) {
  auto kern = gemm_ln_kernel<CL>;
  static bool attr_set = false;
  if (!attr_set) {
    BT_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(GlnCfg::SMEM)));
    attr_set = true;
  }
  const int rbs = (p.M + 127) / 128;
  BT_LAUNCH(kern, dim3(rbs * CL), dim3(GLN_THREADS), GlnCfg::SMEM, s, CL, ta, tb, tr, ty, p);
  return BT_OK;
}

// How many CL-CTA clusters of this kernel the device runs at once (clusters
// must fit inside a GPC: on B200, 22 clusters of 6 but only 15 of 8).
template <int CL>
static int max_active_clusters() {
  static int n = -1;
  if (n < 0) {
    auto kern = gemm_ln_kernel<CL>;
    n = 0;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(GlnCfg::SMEM)) ==
        cudaSuccess) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(CL * 16);
      cfg.blockDim = dim3(GLN_THREADS);
      cfg.dynamicSmemBytes = GlnCfg::SMEM;
      cudaLaunchAttribute a[1];
      a[0].id = cudaLaunchAttributeClusterDimension;
      a[0].val.clusterDim.x = CL;
      a[0].val.clusterDim.y = 1;
      a[0].val.clusterDim.z = 1;
      cfg.attrs = a;
      cfg.numAttrs = 1;
      if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) n = 0;
    }
    (void)cudaGetLastError();
  }
  return n;
}

// Whether the fused kernel applies (N = 128 * CL, CL in {4, 6, 8}) and its
// row blocks fit one wave of clusters.
// Row blocks allowed per resident cluster slot (BT_GEMM_LN_WAVES, default 1).
static int gemm_ln_waves() {
  static int w = -1;
  if (w < 0) {
    const char* e = getenv("BT_GEMM_LN_WAVES");
    w = (e && e[0] >= '1' && e[0] <= '9') ? e[0] - '0' : 1;
  }
  return w;
}

bool gemm_ln_fits(int M, int N, int K) {
  if (N % GLN_BN || K % GLN_BK || K < GLN_BK) return false;
  const int cl = N / GLN_BN;
  const int rbs = (M + 127) / 128;
  const int waves = gemm_ln_waves();
  switch (cl) {
    case 4: return rbs <= waves * max_active_clusters<4>();
    case 6: return rbs <= waves * max_active_clusters<6>();
    case 8: return rbs <= waves * max_active_clusters<8>();
    default: return false;
  }
}

int gemm_ln_launch(const void* A, const void* Bt, const float* bias, const void* residual, const float* gamma,
                   const float* beta, float eps, void* Y, int M, int N, int K, cudaStream_t s) {
  BT_REQUIRE(M >= 0 && N > 0 && K > 0, BT_ESHAPE, "gemm_ln: bad shape M=%d N=%d K=%d", M, N, K);
  BT_REQUIRE(K % GLN_BK == 0, BT_ESHAPE, "gemm_ln: K=%d must be a multiple of 64", K);
  BT_REQUIRE(N % GLN_BN == 0 && (N / GLN_BN == 4 || N / GLN_BN == 6 || N / GLN_BN == 8), BT_ESHAPE,
             "gemm_ln: N=%d must be 512, 768 or 1024", N);
  BT_REQUIRE(bias && gamma && beta && residual && A && Bt && Y, BT_ESHAPE, "gemm_ln: null pointer");
  BT_REQUIRE(eps > 0.f, BT_ESHAPE, "gemm_ln: eps must be > 0");
  if (M == 0) return BT_OK;
  CUtensorMap ta, tb, tr, ty;
  BT_TRY(make_tmap_bf16_2d(&ta, A, M, K, K, 128, GLN_BK));
  BT_TRY(make_tmap_bf16_2d(&tb, Bt, N, K, K, GLN_BN, GLN_BK));
  BT_TRY(make_tmap_bf16_2d(&tr, residual, M, N, N, 128, 64));
  BT_TRY(make_tmap_bf16_2d(&ty, Y, M, N, N, 32, 64));
  GlnParams p;
  p.M = M;
  p.N = N;
  p.K = K;
  p.num_k = K / GLN_BK;
  p.bias = bias;
  p.gamma = gamma;
  p.beta = beta;
  p.eps = eps;
  switch (N / GLN_BN) {
    case 4: return launch_gln<4>(ta, tb, tr, ty, p, s);
    case 6: return launch_gln<6>(ta, tb, tr, ty, p, s);
    default: return launch_gln<8>(ta, tb, tr, ty, p, s);
  }
}

}  // namespace bt

extern "C" int bt_gemm_bias_residual_ln(const void* A, const void* Bt, const float* bias, const void* residual,
                                        const float* gamma, const float* beta, float eps, void* out, int M, int N,
                                        int K, bt_stream_t stream) {
  return bt::gemm_ln_launch(A, Bt, bias, residual, gamma, beta, eps, out, M, N, K, bt::as_stream(stream));
}
