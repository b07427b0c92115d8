/*
 * bt200 -- C ABI of the B200-native (sm_100a) padding-free BERT encoder forward.
 *
 * Every entry point takes plain device pointers owned by the caller, sizes,
 * and a cudaStream_t passed as `bt_stream_t` (void*).  All work is
 * stream-ordered; no entry point synchronises the host except where noted.
 * No torch (or any framework) type crosses this boundary.
 *
 * Each entry replaces one function of the reference package `packbert`
 * (/root/reference/pkg/src/packbert, cited as file:line below); the Python
 * host layer `paper_2210_03052_b200` binds these symbols with ctypes and
 * mirrors the reference's names, argument meaning and error types on top.
 *
 * Return codes: BT_OK (0) or a negative BT_E* code; bt_last_error() returns a
 * thread-local message for the last failure on the calling thread.  The
 * Python layer maps BT_ESHAPE -> ShapeError, BT_ECONFIG -> ConfigError
 * (reference errors.py:8-13).
 */
#ifndef BT200_H
#define BT200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BT_OK 0
#define BT_ESHAPE (-1)  /* operand shapes violate the op's contract       */
#define BT_ECONFIG (-2) /* unsupported model geometry / parameters        */
#define BT_ECUDA (-3)   /* CUDA runtime / driver error                    */
#define BT_EDATA (-4)   /* device-side validation failed (e.g. bad mask)  */

#define BT_F32 0
#define BT_BF16 1

/* GEMM epilogues (reference tensor.py:74-106 EpilogueKind) */
#define BT_EPI_NONE 0          /* C = A B                                   */
#define BT_EPI_BIAS 1          /* C = A B + bias[n]                         */
#define BT_EPI_BIAS_GELU 2     /* C = gelu_tanh(A B + bias[n]) fusion.py:30 */
#define BT_EPI_BIAS_RESIDUAL 3 /* C = (A B + residual) + bias[n]            */

typedef void* bt_stream_t; /* cudaStream_t */

#if defined(__GNUC__)
#define BT_API __attribute__((visibility("default")))
#else
#define BT_API
#endif

/* ---- library ---------------------------------------------------------- */
BT_API int bt_version(void);
BT_API const char* bt_last_error(void);
/* Number of kernels this library has launched since load (process-wide). */
BT_API long long bt_launch_count(void);
/* Number of SMs of the current device (0 if no device). */
BT_API int bt_num_sms(void);

/* ---- packing (packing.py) --------------------------------------------- */

/* compute_plan (packing.py:96-119) on a device mask uint8[bs, mx].
 * Writes lengths[bs], seq_starts[bs+1] (exclusive prefix sum) and
 * offsets[T] (flat padded row of each packed row).  `offsets` must hold
 * bs*mx entries (T is not known before the scan).  *status_dev is set to a
 * bit mask: 1 = entry not in {0,1}, 2 = row not prefix-shaped, 4 = empty row
 * (all three raise ShapeError in the reference, packing.py:103-109 and
 * SeqLengths:27-36).  valid_cnt_dev[0] receives T.                        */
BT_API int bt_plan_mask(const uint8_t* mask, int bs, int mx, int32_t* lengths, int32_t* seq_starts,
                 int32_t* offsets, int32_t* valid_cnt_dev, int32_t* status_dev, bt_stream_t stream);

/* plan_for_lengths (packing.py:122): the same plan from device lengths[bs]
 * (1 <= len <= mx is the caller's contract; validated on the host). */
BT_API int bt_plan_lengths(const int32_t* lengths, int bs, int mx, int32_t* seq_starts, int32_t* offsets,
                    bt_stream_t stream);

/* pack (packing.py:141-148): packed[j, :] = padded[offsets[j], :] (any k >= 1), with an
 * optional fp32 -> bf16 conversion (in/out dtype BT_F32 or BT_BF16).  */
BT_API int bt_pack(const void* padded, int in_dtype, const int32_t* offsets, int T, int k, void* packed,
            int out_dtype, bt_stream_t stream);

/* unpack (packing.py:151-160): padded[b*mx + j, :] = packed[seq_starts[b] + j, :]
 * for j < len[b]; every other padded row is written with exact zeros.  */
BT_API int bt_unpack(const void* packed, int in_dtype, const int32_t* seq_starts, int bs, int mx, int k,
              void* padded, int out_dtype, bt_stream_t stream);

/* ---- GEMM (tensor.py:177-200 gemm + EpilogueHook) ----------------------- */

/* C[M,N] (bf16, row-major, ldc = N) = epilogue(A[M,K] (bf16 row-major) x W)
 * where W is given TRANSPOSED as Bt[N,K] (bf16 row-major, i.e. K-major), the
 * layout the weight cache uploads once (encoder.py:134-150 stores W as
 * [in,out]).  bias is fp32[N]; residual bf16[M,N].  K % 64 == 0, N % 64 == 0.
 * tcgen05/TMEM kernel fed by TMA (sm_100a).  */
BT_API int bt_gemm(const void* A, const void* Bt, const float* bias, const void* residual, void* C, int M, int N,
            int K, int epilogue, bt_stream_t stream);

/* ---- fused variable-length MHA (attention.py:177-314) ------------------- */

/* qkv: bf16 [T, 3*H*d] packed rows, Q|K|V column blocks with their biases
 * already applied (the QKV GEMM epilogue adds them; the reference adds them
 * on operand load, attention.py:209-214 -- same values).  out: bf16 [T, H*d].
 * Dispatch rule of dispatch_mha (attention.py:309-314): the short
 * (tile-resident) kernel iff mx <= cutoff, else the long (streamed,
 * grouped-by-length) kernel.  d must be 64; the short kernel holds up to
 * 384 keys on chip, so cutoff > 384 routes 384 < mx <= cutoff to the long
 * kernel.  split_seq_len is accepted for API parity (the q tile is 128 rows
 * on the tensor cores; the per-row math does not depend on it,
 * attention.py:185-190).  */
BT_API int bt_mha_varlen(const void* qkv, const int32_t* seq_starts, int bs, int mx, int H, int d, int cutoff,
                  int split_seq_len, void* out, int T, bt_stream_t stream);

/* mha_baseline (attention.py:135-174): the same attention over the PADDED
 * layout, qkv bf16 [bs*mx, 3*H*d] (biases applied), out bf16 [bs*mx, H*d].
 * The whole mx x mx rectangle is computed (the unfused baseline's cost),
 * keys >= len[b] are masked out of the softmax and query rows >= len[b] are
 * written as zeros.  seq_starts supplies the lengths. */
BT_API int bt_mha_padded(const void* qkv, const int32_t* seq_starts, int bs, int mx, int H, int d, void* out,
                         bt_stream_t stream);

/* ---- add-bias + residual + LayerNorm (fusion.py:79-98) ----------------- */

/* out = LN((x + residual) + bias) * gamma + beta, row-wise over k columns,
 * population variance, eps as given (reference default 1e-12).
 * x, residual, out: bf16 [T,k] (residual may be NULL -> 0); bias, gamma,
 * beta: fp32 [k] (bias may be NULL).  k % 8 == 0, k <= 4096.  */
BT_API int bt_ln_bias_residual(const void* x, const void* residual, const float* bias, const float* gamma,
                        const float* beta, float eps, void* out, int T, int k, bt_stream_t stream);

/* MHA work schedule for a plan, in a device buffer of bt_plan_sched_bytes(bs, mx) bytes:
 * sched[bs] int2 (start row, length) of the sequences ordered by descending 128-key block count,
 * so the fused MHA dispatches the longest problems first, followed by the same order's list of
 * 128-row query-tile units (and a claim queue) that the MHA's tile-list mode walks for launches of
 * many waves. */
BT_API int bt_plan_sched(const int32_t* seq_starts, int bs, int mx, void* sched, bt_stream_t stream);
BT_API size_t bt_plan_sched_bytes(int bs, int mx);
/* What bt_encoder_forward runs: plan_for_lengths' seq_starts (packing.py:122) and the
 * bt_plan_sched schedule in ONE single-CTA launch; sched holds bt_plan_sched_bytes(bs, mx). */
BT_API int bt_plan_forward(const int32_t* lengths, int bs, int mx, int32_t* seq_starts, void* sched,
                           bt_stream_t stream);
/* pack (packing.py:141) of an fp32 padded batch [bs*mx, k] into bf16 packed rows [T, k], addressed
 * by seq_starts instead of an offsets array (k % 8 == 0). */
BT_API int bt_pack_starts(const float* padded, const int32_t* seq_starts, int bs, int mx, int k, void* packed_bf16,
                          bt_stream_t stream);
/* What bt_encoder_forward runs in front of the layers (one launch, bs <= 4096, k % 8 == 0): the plan
 * (packing.py:96-123 seq_starts + the bt_plan_sched schedule) and pack (packing.py:141-148, fp32 ->
 * bf16) of the valid rows.  x_padded non-NULL: padded input [bs*mx, k]; row_map[T] receives each packed
 * row's padded row index (offsets, packing.py:123) and out_padded's padded rows are set to exact zeros
 * (packing.py:158-159; bt_ln_bias_residual_out later writes the valid rows).  x_padded NULL: the input
 * x_packed_in [T, k] is already packed (out_padded / row_map unused).  sched holds
 * bt_plan_sched_bytes(bs, mx) bytes. */
BT_API int bt_forward_prologue(const int32_t* lengths, int bs, int mx, int k, const float* x_padded,
                               const float* x_packed_in, void* x_packed_bf16, int32_t* seq_starts, void* sched,
                               float* out_padded, int32_t* row_map, int T, bt_stream_t stream);
/* bt_ln_bias_residual whose rows go to an fp32 output: out_f32[row_map[r]] (row r itself when row_map
 * is NULL) = the bf16-rounded LayerNorm row widened to fp32 -- the forward's last LayerNorm fused with
 * unpack (packing.py:151-160). */
BT_API int bt_ln_bias_residual_out(const void* x, const void* residual, const float* bias, const float* gamma,
                                   const float* beta, float eps, float* out_f32, const int32_t* row_map, int T,
                                   int k, bt_stream_t stream);
/* 1 when bt_encoder_forward runs bt_forward_prologue + bt_ln_bias_residual_out at its ends (else
 * bt_plan_forward + bt_pack_starts ... bt_unpack). */
BT_API int bt_one_launch_ends(int k, int bs);
/* bt_mha_varlen with the CTA order of a bt_plan_sched schedule (what bt_encoder_forward runs). */
BT_API int bt_mha_varlen_sched(const void* qkv, const int32_t* seq_starts, const void* sched, int bs, int mx, int H,
                               int d, int cutoff, void* out, int T, bt_stream_t stream);

/* 1 if bt_encoder_layer / bt_encoder_forward use bt_gemm_bias_residual_ln after the attention-output
 * projection for T tokens of hidden size k (else GEMM + bt_ln_bias_residual). */
BT_API int bt_fused_attn_out_ln(int T, int k);
/* 1 if bt_encoder_layer / bt_encoder_forward use bt_gemm_bias_residual_ln after the FFN2 projection
 * (encoder.py:404-407) for T tokens, hidden size k and FFN width f -- every layer except the last of a
 * forward that ends in bt_ln_bias_residual_out (bt_one_launch_ends). */
BT_API int bt_fused_ffn2_ln(int T, int k, int f);

/* Fused attention-output / FFN2 projection + add-bias + residual + LayerNorm (encoder.py:385-388 and
 * :404-407, i.e. gemm then fusion.py:79 add_bias_residual_layernorm):
 *   out[M,N] = LN((A[M,K] Bt[N,K]^T + residual) + bias) * gamma + beta,  bf16 in / out, fp32 math.
 * N in {512, 768, 1024}; one row block per thread-block cluster of N/128 CTAs (row statistics combined
 * through distributed shared memory). */
BT_API int bt_gemm_bias_residual_ln(const void* A, const void* Bt, const float* bias, const void* residual,
                                    const float* gamma, const float* beta, float eps, void* out, int M, int N,
                                    int K, bt_stream_t stream);

/* ---- element-wise passes (fusion.py:23-76; unfused ladder variants) ---- */

/* out[r, c] = act(x[r, c] + bias[c]) for r < rows, c < cols (act 0 = none,
 * 1 = tanh-GELU, fusion.py:23-35); row pitches ldx / ldo in elements so a
 * column slice of a wider tensor can be read or written.  bias may be NULL. */
BT_API int bt_bias_act(const void* x, int in_dtype, int ldx, const float* bias, void* out, int out_dtype, int ldo,
                       int rows, int cols, int act, bt_stream_t stream);

/* out = x + y over n elements (n % 8 == 0), fusion.py:66-69. */
BT_API int bt_add(const void* x, const void* y, void* out, int dtype, long long n, bt_stream_t stream);

/* ---- encoder (encoder.py:337-437) --------------------------------------- */

typedef struct bt_layer_weights {
  const void* qkv_w;  /* bf16 [3k, k]  (qkv_weight^T)            */
  const float* qkv_b; /* fp32 [3k]                                */
  const void* ao_w;   /* bf16 [k, k]   (attn_out_weight^T)       */
  const float* ao_b;  /* fp32 [k]                                 */
  const void* w1;     /* bf16 [f, k]   (ffn_w1^T), f = ffn*k     */
  const float* b1;    /* fp32 [f]                                 */
  const void* w2;     /* bf16 [k, f]   (ffn_w2^T)                */
  const float* b2;    /* fp32 [k]                                 */
  const float* ln0_g; /* fp32 [k] */
  const float* ln0_b; /* fp32 [k] */
  const float* ln1_g; /* fp32 [k] */
  const float* ln1_b; /* fp32 [k] */
  float ln0_eps;
  float ln1_eps;
} bt_layer_weights;

typedef struct bt_layer_cfg {
  int head_num;
  int head_size;
  int ffn_scale;
  int max_seq_len;
  int cutoff;
  int split_seq_len;
} bt_layer_cfg;

/* Scratch bytes bt_encoder_layer needs for T packed rows. */
BT_API size_t bt_layer_workspace_bytes(const bt_layer_cfg* cfg, int T);

/* encoder_layer with OptFlags.all_on() (encoder.py:337-408): x_inout is the
 * packed bf16 [T, k] layer input, overwritten with the layer output. */
BT_API int bt_encoder_layer(const bt_layer_weights* w, const bt_layer_cfg* cfg, const int32_t* seq_starts, int bs,
                     int T, void* x_inout, void* ws, size_t ws_bytes, bt_stream_t stream);

/* Scratch bytes bt_encoder_forward needs (plan + packed activations + layer scratch). */
BT_API size_t bt_forward_workspace_bytes(const bt_layer_cfg* cfg, int bs, int T);

/* forward (encoder.py:411-437): lengths (int32[bs]) -> plan ->
 * pack(x_padded fp32 [bs*mx, k]) -> n_layers x encoder_layer -> unpack to
 * out_padded fp32 [bs*mx, k] with exact-zero padded rows.  `layers` is a
 * HOST array of n_layers weight structs (repeat one struct for ALBERT-style
 * sharing, encoder.py:130-131).  T = sum(lengths) must be supplied by the
 * caller (it is known on the host; no device->host sync happens).
 * lengths, x_padded and out_padded may be device memory or pinned
 * (page-locked, UVA-mapped) HOST memory: the pack kernel then gathers only
 * the valid input rows straight from host memory over PCIe and the unpack
 * kernel writes the padded output straight into host memory -- the
 * end-to-end path needs no separate bulk H2D / D2H copies.  */
BT_API int bt_encoder_forward(const bt_layer_weights* layers, int n_layers, const bt_layer_cfg* cfg,
                       const int32_t* lengths, int bs, int T, const float* x_padded, float* out_padded,
                       void* ws, size_t ws_bytes, bt_stream_t stream);

/* ---- test hooks (exercise every kernel instantiation) ------------------ */
/* bt_gemm with a forced tile: bn in {64,128,256} = one CTA 128 x bn, bn in {-64,-128,-192,-256} = SM pair (cta_group::2) 256 x |bn|. */
BT_API int bt_gemm_bn(const void* A, const void* Bt, const float* bias, const void* residual, void* C, int M, int N,
                      int K, int epilogue, int bn, bt_stream_t stream);
/* bt_mha_varlen forcing the short (path = 1, mx <= 384) or long (path = 2) kernel. */
BT_API int bt_mha_varlen_path(const void* qkv, const int32_t* seq_starts, int bs, int mx, int H, int d, void* out,
                              int T, int path, bt_stream_t stream);

/* Debug hook: per-CTA globaltimer event trace of the GEMM kernels (64 u64
 * slots per CTA, see csrc/gemm_sm100.cu); NULL turns tracing off. */
BT_API int bt_debug_gemm_trace(unsigned long long* buf);
/* Debug hook: 0 normal, 1 = GEMMs skip the MMAs, 2 = GEMMs skip the TMA loads, 3 / 4 / 5 = stream-K
 * off / on / automatic, 6 / 7 / 8 = epilogue probes: no output store / no TMEM loads / TMEM loads only
 * (results invalid in 1, 2, 6, 7, 8). */
BT_API int bt_debug_gemm_mode(int mode);
/* Debug hook: install n cudaEvent_t (as void*) that the next bt_encoder_forward records after each
 * launch group: [0] start, [1] plan + pack, 7 per layer, then unpack; NULL uninstalls. */
BT_API int bt_debug_forward_events(void** events, int n);
/* Test hook: query tiles per fused-MHA CTA (0 = automatic: 4 for launches of many waves, else 1). */
BT_API int bt_debug_mha_qg(int qg);
/* Test hook: the MHA's tile-list mode (bt_mha_varlen_sched / the forward): 0 off,
 * 1 automatic (launches of many waves), 2 always, -1 the
 * BT_MHA_LIST environment policy; grid > 0 pins the number of CTAs walking the list. */
BT_API int bt_debug_mha_list(int mode, int grid);
/* Test hook: the MHA's segment kernel (bt_mha_varlen_sched / the forward, batches of bs <= 256 and
 * max_seq_len <= 256: adjacent sequences of <= 128 rows share one CTA per head, rows masked to their
 * own sequence): 0 off, 1 or 2 on, -1 the BT_MHA_SEG environment policy (default on). */
BT_API int bt_debug_mha_seg(int mode);
/* Debug hook: resident CTAs per SM of an MHA variant (0 short/2 blocks, 1 short/3 blocks, 2 long,
 * 3 multi-tile long); info[3] (optional) receives registers, static and max dynamic smem. */
BT_API int bt_debug_mha_occupancy(int which, int* info);
/* Debug hook: per-CTA globaltimer event trace of the MHA kernels (32 u64 slots per CTA). */
BT_API int bt_debug_mha_trace(unsigned long long* buf);

/* Instrumented FlopCounter (replaces the counter.add calls of reference
 * tensor.py:198-199 / attention.py:232-236 with launch-level counting).
 * bt_flops_enable(dev): from now on every GEMM the encoder layer launches adds
 * 2*M*N*K of its launch shape under its module key (host counters, read with
 * bt_flops_read: out[0..3] = gemm0 QKV, gemm1 attention output, gemm2 FFN1,
 * gemm3 FFN2), and every MHA tile adds the FLOPs it computed (4*d per query
 * row x key of its problem) to the device u64 *dev.  NULL turns it off. */
BT_API int bt_flops_enable(unsigned long long* dev_mha_counter);
BT_API int bt_flops_read(long long* out4);

/* forward on the packed layout: x_packed / out_packed fp32 [T, k] (device).
 * Same pipeline as bt_encoder_forward minus the gather / scatter; the
 * end-to-end host path DMAs only valid rows in and out (bt_copy_rows). */
BT_API int bt_encoder_forward_packed(const bt_layer_weights* layers, int n_layers, const bt_layer_cfg* cfg,
                                     const int32_t* lengths, int bs, int T, const float* x_packed, float* out_packed,
                                     void* ws, size_t ws_bytes, bt_stream_t stream);

/* pack / unpack as DMA: copy each sequence's valid rows between a padded
 * buffer [bs*mx, row_bytes] and a packed one [T, row_bytes] with async
 * cudaMemcpy (host or device memory on either side; lengths_host on the
 * host).  to_packed = 1: padded -> packed, 0: packed -> padded (padded rows
 * untouched). */
BT_API int bt_copy_rows(void* dst, const void* src, const int32_t* lengths_host, int bs, int mx, long long row_bytes,
                        int to_packed, bt_stream_t stream);

/* test hook: the four-CTAs-per-SM fused MHA (64-key blocks, P over S in TMEM)
 * on (1) / off (0) for the packed launches outside the segment kernel; -1
 * restores the BT_MHA64 policy (default on). */
BT_API int bt_debug_mha64(int mode);

/* page-locked host staging memory for pageable inputs (the reference's numpy
 * Tensor): write_combined = 1 allocates it write-combined, so the CPU's
 * staging stores bypass its caches and the following DMA reads at the PCIe
 * rate instead of snooping dirty lines.  *out = NULL on failure. */
BT_API int bt_host_alloc(size_t bytes, int write_combined, void** out);
BT_API int bt_host_free(void* p);

#ifdef __cplusplus
}
#endif
#endif /* BT200_H */
