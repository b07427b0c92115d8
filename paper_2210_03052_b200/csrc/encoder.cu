// Encoder runtime: one post-LN BERT layer and the stacked, padding-free
// forward pass (reference encoder.py:337-437, OptFlags.all_on()), issued
// stream-ordered from the host with no synchronisation, so the whole forward
// can be captured into one CUDA graph.
//
// Layer data flow (packed [T, *] bf16 activations):
//   qkv  = x Wqkv + bqkv                     GEMM #0 (bias epilogue)
//   ctx  = fused varlen MHA(qkv)             short / long path
//   proj = ctx Wo                            GEMM #1
//   y0   = LN((proj + x) + bo)               fused add-bias+residual+LN
//   h1   = gelu(y0 W1 + b1)                  GEMM #2 (bias+GELU epilogue)
//   h2   = h1 W2                             GEMM #3
//   x    = LN((h2 + y0) + b2)                fused add-bias+residual+LN

#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace bt {
int gemm_launch(const void* A, const void* Bt, const float* bias, const void* residual, void* C, int M, int N, int K,
                int epi, int force_bn, cudaStream_t s);
int mha_launch(const void* qkv, const int32_t* seq_starts, int bs, int mx, int H, int d, int cutoff, int T, void* out,
               int force_path, cudaStream_t s, int padded, const void* sched);
bool gemm_ln_fits(int M, int N, int K);
int ln_launch(const void* x, const void* residual, const float* bias, const float* gamma, const float* beta, float eps,
              void* out, int T, int k, cudaStream_t s, float* outf, const int32_t* row_map);
int gemm_ln_launch(const void* A, const void* Bt, const float* bias, const void* residual, const float* gamma,
                   const float* beta, float eps, void* Y, int M, int N, int K, cudaStream_t s);
// BT_FUSED_LN: 0 = GEMM + separate LayerNorm kernel everywhere, 1 = the
// fused GEMM+LN kernel after the attention-output GEMM (K = k), 2 (default) =
// after both projections (each where gemm_ln_fits: one wave of clusters).  The
// forward's last layer keeps FFN2 + the LayerNorm that writes the fp32 output
// rows (one-launch ends).  Round 1 measured mode 2 slower at C2 (0.809 vs
// 0.787 ms/step); after the GEMM+LN kernel's deeper weight prefetch and the
// GEMM changes it is faster: C2 0.685 vs 0.700 ms/step (three alternations,
// scripts/ab_gemm_ln_ffn2.sh); C3's row blocks exceed one wave (unchanged).
static int fused_ln_mode() {
  static int mode = -1;
  if (mode < 0) {
    const char* e = getenv("BT_FUSED_LN");
    mode = (e && e[0] >= '0' && e[0] <= '2') ? e[0] - '0' : 2;
  }
  return mode;
}


// FFN2 + LN1 fusion: one wave of clusters, and at least 8 row blocks -- with
// fewer, the 128 x 128 tiles over K = 4k leave most SMs idle and the plain
// SM-pair GEMM + LN is as fast or faster (graph-captured BERT-base, same box:
// bs 1 x mx 1024 (T 614) 0.667 vs 0.608 ms, bs 1 x 64 (T 38) 0.456 vs 0.437,
// bs 16 x 64 (T 614) 0.493 vs 0.486; at C2 (T 2458) 0.685 vs 0.700).
static bool fused_ffn2_ln(int T, int k, int f) {
  return fused_ln_mode() >= 2 && T > 7 * 128 && gemm_ln_fits(T, k, f);
}

// Diagnostics only (results are wrong when set): BT_DEBUG_SKIP = a set of
// letters naming launches of every layer to leave out -- q (QKV GEMM), m
// (MHA), a (attn-out GEMM + LN0), f (FFN1), s (FFN2), l (LN1) -- to measure
// each launch's cost inside the graph-replayed step by difference.
static bool debug_skip(char c) {
  static const char* e = getenv("BT_DEBUG_SKIP");
  return e && strchr(e, c) != nullptr;
}

static inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// The forward's ends as one prologue launch (plan + pack + zeroing of padded
// output rows) and a last LayerNorm that writes the fp32 output rows itself
// (no unpack).  BT_ONE_LAUNCH_ENDS=0 restores plan_forward + pack_starts +
// unpack (A/B); the fused FFN2+LN mode and very large batches use them too.
static bool one_launch_ends(int k, int bs) {
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("BT_ONE_LAUNCH_ENDS");
    env = (e && e[0] == '0') ? 0 : 1;
  }
  return env == 1 && k % 8 == 0 && bs <= 4096 && !debug_skip('l');
}

// Instrumented FlopCounter (reference tensor.py:198-199, attention.py:232-236):
// while enabled, every GEMM the layer launches adds 2*M*N*K under its module
// key (gemm0 QKV, gemm1 attention output, gemm2 FFN1, gemm3 FFN2) from the
// shapes it was launched with, and the MHA kernel adds the work its tiles did
// to a device counter.  Off by default (no cost on the hot path).
extern unsigned long long* g_mha_flops;
static bool g_flops_on = false;
static long long g_flops[4] = {0, 0, 0, 0};
static void count_gemm(int key, int M, int N, int K) {
  if (g_flops_on) g_flops[key] += 2LL * M * N * K;
}

struct LayerWs {
  __nv_bfloat16 *qkv, *ctx, *proj, *y0, *h1;
};

static size_t layer_ws_bytes(int k, int f, int T) {
  const size_t t = static_cast<size_t>(T);
  return align_up(t * 3 * k * 2) + 3 * align_up(t * k * 2) + align_up(t * f * 2);
}

static LayerWs carve_layer(void* ws, int k, int f, int T) {
  const size_t t = static_cast<size_t>(T);
  uint8_t* p = static_cast<uint8_t*>(ws);
  LayerWs w;
  w.qkv = reinterpret_cast<__nv_bfloat16*>(p);
  p += align_up(t * 3 * k * 2);
  w.ctx = reinterpret_cast<__nv_bfloat16*>(p);
  p += align_up(t * k * 2);
  w.proj = reinterpret_cast<__nv_bfloat16*>(p);
  p += align_up(t * k * 2);
  w.y0 = reinterpret_cast<__nv_bfloat16*>(p);
  p += align_up(t * k * 2);
  w.h1 = reinterpret_cast<__nv_bfloat16*>(p);
  return w;
}

static int check_cfg(const bt_layer_cfg* cfg) {
  BT_REQUIRE(cfg != nullptr, BT_ECONFIG, "null layer config");
  BT_REQUIRE(cfg->head_num >= 1 && cfg->head_size >= 1 && cfg->ffn_scale >= 1 && cfg->max_seq_len >= 1, BT_ECONFIG,
             "layer config fields must be >= 1");
  BT_REQUIRE(cfg->head_size == 64, BT_ECONFIG, "the sm_100a kernels support head_size 64, got %d", cfg->head_size);
  BT_REQUIRE(cfg->split_seq_len >= 1, BT_ECONFIG, "split_seq_len must be >= 1, got %d", cfg->split_seq_len);
  return BT_OK;
}

}  // namespace bt

extern "C" int bt_ln_bias_residual(const void* x, const void* residual, const float* bias, const float* gamma,
                                   const float* beta, float eps, void* out, int T, int k, bt_stream_t stream);
extern "C" int bt_pack(const void*, int, const int32_t*, int, int, void*, int, bt_stream_t);
extern "C" int bt_unpack(const void*, int, const int32_t*, int, int, int, void*, int, bt_stream_t);
extern "C" int bt_plan_lengths(const int32_t*, int, int, int32_t*, int32_t*, bt_stream_t);
extern "C" int bt_plan_sched(const int32_t*, int, int, void*, bt_stream_t);
extern "C" int bt_bias_act(const void*, int, int, const float*, void*, int, int, int, int, int, bt_stream_t);


extern "C" size_t bt_layer_workspace_bytes(const bt_layer_cfg* cfg, int T) {
  if (!cfg) return 0;
  const int k = cfg->head_num * cfg->head_size;
  return bt::layer_ws_bytes(k, cfg->ffn_scale * k, T < 1 ? 1 : T);
}

namespace bt {
// Debug hook (bt_debug_forward_events): when installed, the forward records
// events[i] after each of its launches (plan/pack, then 7 per layer), so a
// caller can attribute device time per kernel inside a real forward.
static cudaEvent_t* g_fwd_events = nullptr;
static int g_fwd_events_n = 0;
static int g_fwd_event_idx = 0;
static int mark(cudaStream_t s) {
  if (g_fwd_events && g_fwd_event_idx < g_fwd_events_n) BT_CUDA_CHECK(cudaEventRecord(g_fwd_events[g_fwd_event_idx++], s));
  return BT_OK;
}
// One post-LN layer.
// `sched` (optional): the MHA work schedule of the batch (bt_plan_sched).
static int encoder_layer_impl(const bt_layer_weights* w, const bt_layer_cfg* cfg, const int32_t* seq_starts, int bs,
                              int T, void* x_inout, void* ws, size_t ws_bytes, bt_stream_t stream,
                              const void* sched = nullptr, float* final_out = nullptr,
                              const int32_t* row_map = nullptr) {
  BT_TRY(bt::check_cfg(cfg));
  BT_REQUIRE(w != nullptr, BT_ESHAPE, "null layer weights");
  BT_REQUIRE(T >= 1 && bs >= 1, BT_ESHAPE, "encoder_layer: T=%d bs=%d", T, bs);
  const int k = cfg->head_num * cfg->head_size;
  const int f = cfg->ffn_scale * k;
  BT_REQUIRE(ws_bytes >= bt::layer_ws_bytes(k, f, T), BT_ESHAPE, "encoder_layer: workspace too small (%zu < %zu)",
             ws_bytes, bt::layer_ws_bytes(k, f, T));
  cudaStream_t s = bt::as_stream(stream);
  bt::LayerWs L = bt::carve_layer(ws, k, f, T);
  auto* x = static_cast<__nv_bfloat16*>(x_inout);

  if (!debug_skip('q')) BT_TRY(bt::gemm_launch(x, w->qkv_w, w->qkv_b, nullptr, L.qkv, T, 3 * k, k, BT_EPI_BIAS, 0, s));
  count_gemm(0, T, 3 * k, k);
  BT_TRY(mark(s));
  if (!debug_skip('m'))
    BT_TRY(bt::mha_launch(L.qkv, seq_starts, bs, cfg->max_seq_len, cfg->head_num, cfg->head_size, cfg->cutoff, T,
                          L.ctx, 0, s, 0, sched));
  BT_TRY(mark(s));
  if (debug_skip('a')) {
  } else if (fused_ln_mode() >= 1 && gemm_ln_fits(T, k, k)) {  // y0 = LN((ctx Wo + x) + bo), one kernel
    BT_TRY(gemm_ln_launch(L.ctx, w->ao_w, w->ao_b, x, w->ln0_g, w->ln0_b, w->ln0_eps, L.y0, T, k, k, s));
    count_gemm(1, T, k, k);
    BT_TRY(mark(s));
  } else {
    BT_TRY(bt::gemm_launch(L.ctx, w->ao_w, nullptr, nullptr, L.proj, T, k, k, BT_EPI_NONE, 0, s));
    count_gemm(1, T, k, k);
    BT_TRY(mark(s));
    BT_TRY(bt_ln_bias_residual(L.proj, x, w->ao_b, w->ln0_g, w->ln0_b, w->ln0_eps, L.y0, T, k, stream));
  }
  BT_TRY(mark(s));
  if (!debug_skip('f')) BT_TRY(bt::gemm_launch(L.y0, w->w1, w->b1, nullptr, L.h1, T, f, k, BT_EPI_BIAS_GELU, 0, s));
  count_gemm(2, T, f, k);
  BT_TRY(mark(s));
  if (fused_ffn2_ln(T, k, f) && final_out == nullptr) {  // x = LN((h1 W2 + y0) + b2), one kernel
    BT_TRY(gemm_ln_launch(L.h1, w->w2, w->b2, L.y0, w->ln1_g, w->ln1_b, w->ln1_eps, x, T, k, f, s));
    count_gemm(3, T, k, f);
    BT_TRY(mark(s));
  } else {
    if (!debug_skip('s')) BT_TRY(bt::gemm_launch(L.h1, w->w2, nullptr, nullptr, L.proj, T, k, f, BT_EPI_NONE, 0, s));
    count_gemm(3, T, k, f);
    BT_TRY(mark(s));
    // (final_out: the forward's last layer writes its output rows as fp32
    // straight into the caller's output -- padded rows via row_map -- instead
    // of x + an unpack pass)
    if (!debug_skip('l'))
      BT_TRY(bt::ln_launch(L.proj, L.y0, w->b2, w->ln1_g, w->ln1_b, w->ln1_eps, final_out ? nullptr : x, T, k, s,
                           final_out, row_map));
  }
  BT_TRY(mark(s));
  return BT_OK;
}
}  // namespace bt

extern "C" int bt_one_launch_ends(int k, int bs) { return bt::one_launch_ends(k, bs) ? 1 : 0; }

// 1 when the forward fuses the attention-output GEMM with add-bias + residual
// + LayerNorm for this token count and hidden size (bench / tooling query).
extern "C" int bt_fused_attn_out_ln(int T, int k) {
  return (bt::fused_ln_mode() >= 1 && bt::gemm_ln_fits(T, k, k)) ? 1 : 0;
}

// 1 when the forward fuses the FFN2 GEMM with add-bias + residual + LayerNorm
// (every layer but a one-launch-ends forward's last) for T tokens.
extern "C" int bt_fused_ffn2_ln(int T, int k, int f) { return bt::fused_ffn2_ln(T, k, f) ? 1 : 0; }

extern "C" int bt_encoder_layer(const bt_layer_weights* w, const bt_layer_cfg* cfg, const int32_t* seq_starts, int bs,
                                int T, void* x_inout, void* ws, size_t ws_bytes, bt_stream_t stream) {
  return bt::encoder_layer_impl(w, cfg, seq_starts, bs, T, x_inout, ws, ws_bytes, stream);
}

extern "C" size_t bt_forward_workspace_bytes(const bt_layer_cfg* cfg, int bs, int T) {
  if (!cfg) return 0;
  const int k = cfg->head_num * cfg->head_size;
  const size_t t = static_cast<size_t>(T < 1 ? 1 : T);
  return bt::align_up((bs + 1) * sizeof(int32_t)) + bt::align_up(bt::sched_bytes(bs, cfg->max_seq_len)) +
         bt::align_up(t * sizeof(int32_t)) +
         bt::align_up(t * k * 2) + bt_layer_workspace_bytes(cfg, T);
}

extern "C" int bt_encoder_forward(const bt_layer_weights* layers, int n_layers, const bt_layer_cfg* cfg,
                                  const int32_t* lengths, int bs, int T, const float* x_padded, float* out_padded,
                                  void* ws, size_t ws_bytes, bt_stream_t stream) {
  BT_TRY(bt::check_cfg(cfg));
  BT_REQUIRE(n_layers >= 1 && layers != nullptr, BT_ECONFIG, "need >= 1 layer");
  BT_REQUIRE(bs >= 1 && T >= 1 && T <= bs * cfg->max_seq_len, BT_ESHAPE, "forward: bs=%d T=%d mx=%d", bs, T,
             cfg->max_seq_len);
  BT_REQUIRE(ws_bytes >= bt_forward_workspace_bytes(cfg, bs, T), BT_ESHAPE, "forward: workspace too small");
  const int k = cfg->head_num * cfg->head_size;
  const int mx = cfg->max_seq_len;
  uint8_t* p = static_cast<uint8_t*>(ws);
  auto* seq_starts = reinterpret_cast<int32_t*>(p);
  p += bt::align_up((bs + 1) * sizeof(int32_t));
  void* sched = p;
  p += bt::align_up(bt::sched_bytes(bs, mx));
  auto* offsets = reinterpret_cast<int32_t*>(p);
  p += bt::align_up(static_cast<size_t>(T) * sizeof(int32_t));
  void* x = p;
  p += bt::align_up(static_cast<size_t>(T) * k * 2);
  void* lws = p;
  const size_t lws_bytes = bt_layer_workspace_bytes(cfg, T);

  bt::g_fwd_event_idx = 0;
  BT_TRY(bt::mark(bt::as_stream(stream)));
  if (bt::one_launch_ends(k, bs)) {
    // plan + pack + zeroing of the output's padded rows in one launch; the
    // last layer's LayerNorm writes the valid output rows (offsets = row_map)
    BT_TRY(bt_forward_prologue(lengths, bs, mx, k, x_padded, nullptr, x, seq_starts, sched, out_padded, offsets, T,
                            stream));
    BT_TRY(bt::mark(bt::as_stream(stream)));
    for (int li = 0; li < n_layers; ++li)
      BT_TRY(bt::encoder_layer_impl(&layers[li], cfg, seq_starts, bs, T, x, lws, lws_bytes, stream, sched,
                                    li == n_layers - 1 ? out_padded : nullptr, offsets));
    BT_TRY(bt::mark(bt::as_stream(stream)));
    return BT_OK;
  }
  if (k % 8 == 0) {
    BT_TRY(bt_plan_forward(lengths, bs, mx, seq_starts, sched, stream));
    BT_TRY(bt_pack_starts(x_padded, seq_starts, bs, mx, k, x, stream));
  } else {
    BT_TRY(bt_plan_lengths(lengths, bs, mx, seq_starts, offsets, stream));
    BT_TRY(bt_plan_sched(seq_starts, bs, mx, sched, stream));
    BT_TRY(bt_pack(x_padded, BT_F32, offsets, T, k, x, BT_BF16, stream));
  }
  BT_TRY(bt::mark(bt::as_stream(stream)));
  for (int li = 0; li < n_layers; ++li)
    BT_TRY(bt::encoder_layer_impl(&layers[li], cfg, seq_starts, bs, T, x, lws, lws_bytes, stream, sched));
  BT_TRY(bt_unpack(x, BT_BF16, seq_starts, bs, mx, k, out_padded, BT_F32, stream));
  BT_TRY(bt::mark(bt::as_stream(stream)));
  return BT_OK;
}

// Debug hook: install (or clear, with NULL / 0) an array of n cudaEvent_t the
// next bt_encoder_forward records after its launches: [0] start, [1] after
// plan + pack, then 7 per layer (qkv, mha, attn-out, ln0, ffn1, ffn2,
// ln1), then after unpack.
extern "C" int bt_debug_forward_events(void** events, int n) {
  bt::g_fwd_events = reinterpret_cast<cudaEvent_t*>(events);
  bt::g_fwd_events_n = events ? n : 0;
  bt::g_fwd_event_idx = 0;
  return BT_OK;
}

extern "C" int bt_encoder_forward_packed(const bt_layer_weights* layers, int n_layers, const bt_layer_cfg* cfg,
                                         const int32_t* lengths, int bs, int T, const float* x_packed,
                                         float* out_packed, void* ws, size_t ws_bytes, bt_stream_t stream) {
  BT_TRY(bt::check_cfg(cfg));
  BT_REQUIRE(n_layers >= 1 && layers != nullptr, BT_ECONFIG, "need >= 1 layer");
  BT_REQUIRE(bs >= 1 && T >= 1 && T <= bs * cfg->max_seq_len, BT_ESHAPE, "forward_packed: bs=%d T=%d mx=%d", bs, T,
             cfg->max_seq_len);
  BT_REQUIRE(ws_bytes >= bt_forward_workspace_bytes(cfg, bs, T), BT_ESHAPE, "forward_packed: workspace too small");
  const int k = cfg->head_num * cfg->head_size;
  const int mx = cfg->max_seq_len;
  uint8_t* p = static_cast<uint8_t*>(ws);
  auto* seq_starts = reinterpret_cast<int32_t*>(p);
  p += bt::align_up((bs + 1) * sizeof(int32_t));
  void* sched = p;
  p += bt::align_up(bt::sched_bytes(bs, mx));
  p += bt::align_up(static_cast<size_t>(T) * sizeof(int32_t));  // offsets (unused: input already packed)
  void* x = p;
  p += bt::align_up(static_cast<size_t>(T) * k * 2);
  void* lws = p;
  const size_t lws_bytes = bt_layer_workspace_bytes(cfg, T);
  if (bt::one_launch_ends(k, bs)) {
    // plan + fp32 -> bf16 in one launch; the last LayerNorm writes fp32 rows
    BT_TRY(bt_forward_prologue(lengths, bs, mx, k, nullptr, x_packed, x, seq_starts, sched, nullptr, nullptr, T, stream));
    for (int li = 0; li < n_layers; ++li)
      BT_TRY(bt::encoder_layer_impl(&layers[li], cfg, seq_starts, bs, T, x, lws, lws_bytes, stream, sched,
                                    li == n_layers - 1 ? out_packed : nullptr, nullptr));
    return BT_OK;
  }
  BT_TRY(bt_plan_forward(lengths, bs, mx, seq_starts, sched, stream));
  BT_TRY(bt_bias_act(x_packed, BT_F32, k, nullptr, x, BT_BF16, k, T, k, 0, stream));  // fp32 -> bf16
  for (int li = 0; li < n_layers; ++li)
    BT_TRY(bt::encoder_layer_impl(&layers[li], cfg, seq_starts, bs, T, x, lws, lws_bytes, stream, sched));
  BT_TRY(bt_bias_act(x, BT_BF16, k, nullptr, out_packed, BT_F32, k, T, k, 0, stream));  // bf16 -> fp32
  return BT_OK;
}

// Copy the valid rows of each sequence between a padded host / device buffer
// [bs*mx, row_bytes] and a packed one [T, row_bytes] with async DMA copies
// (adjacent sequences that are contiguous on both sides are merged), one
// cudaMemcpyAsync per run.
extern "C" int bt_copy_rows(void* dst, const void* src, const int32_t* lengths_host, int bs, int mx,
                            long long row_bytes, int to_packed, bt_stream_t stream) {
  BT_REQUIRE(bs >= 1 && mx >= 1 && row_bytes > 0 && lengths_host, BT_ESHAPE, "copy_rows: bad arguments");
  cudaStream_t s = bt::as_stream(stream);
  std::vector<void*> dsts, srcs;
  std::vector<size_t> sizes;
  long long packed_row = 0;
  int b = 0;
  while (b < bs) {
    BT_REQUIRE(lengths_host[b] >= 1 && lengths_host[b] <= mx, BT_ESHAPE, "copy_rows: length %d out of range",
               lengths_host[b]);
    const long long padded_row = static_cast<long long>(b) * mx;
    long long rows = lengths_host[b];
    int e = b + 1;
    while (e < bs && lengths_host[e - 1] == mx && lengths_host[e] >= 1) {  // contiguous run
      rows += lengths_host[e];
      ++e;
      if (lengths_host[e - 1] != mx) break;
    }
    const char* s_ptr = static_cast<const char*>(src) + (to_packed ? padded_row : packed_row) * row_bytes;
    char* d_ptr = static_cast<char*>(dst) + (to_packed ? packed_row : padded_row) * row_bytes;
    dsts.push_back(d_ptr);
    srcs.push_back(const_cast<char*>(s_ptr));
    sizes.push_back(static_cast<size_t>(rows * row_bytes));
    packed_row += rows;
    b = e;
  }
  for (size_t i = 0; i < sizes.size(); ++i)
    BT_CUDA_CHECK(cudaMemcpyAsync(dsts[i], srcs[i], sizes[i], cudaMemcpyDefault, s));
  return BT_OK;
}

extern "C" int bt_host_alloc(size_t bytes, int write_combined, void** out) {
  BT_REQUIRE(out != nullptr && bytes > 0, BT_ESHAPE, "host_alloc: bad arguments");
  *out = nullptr;
  BT_CUDA_CHECK(cudaHostAlloc(out, bytes, write_combined ? cudaHostAllocWriteCombined : cudaHostAllocDefault));
  return BT_OK;
}

extern "C" int bt_host_free(void* p) {
  if (p) BT_CUDA_CHECK(cudaFreeHost(p));
  return BT_OK;
}

// Instrumented FLOP counting on (dev_mha_counter: a device u64 the MHA tiles
// add to; the GEMM counts start from zero) or off (NULL).
extern "C" int bt_flops_enable(unsigned long long* dev_mha_counter) {
  bt::g_flops_on = dev_mha_counter != nullptr;
  bt::g_mha_flops = dev_mha_counter;
  for (long long& v : bt::g_flops) v = 0;
  return BT_OK;
}

// The GEMM FLOPs counted since bt_flops_enable: out[0..3] = gemm0..gemm3.
extern "C" int bt_flops_read(long long* out4) {
  BT_REQUIRE(out4 != nullptr, BT_ESHAPE, "bt_flops_read: null output");
  for (int i = 0; i < 4; ++i) out4[i] = bt::g_flops[i];
  return BT_OK;
}
