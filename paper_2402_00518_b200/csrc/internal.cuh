// internal.cuh -- declarations shared by the library's translation units.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdint>
#include <cstdlib>
#include <utility>
#include "gemm.cuh"

namespace ee {

// Launch with programmatic stream serialization (PDL, the decode chain): the
// kernel may start while the previous kernel of the stream drains, so it must
// call griddep_wait() (ptx.cuh) before touching memory that kernel writes or
// reads.  EE_PDL=0 launches normally (A/B).
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("EE_PDL");
    return e ? atoi(e) != 0 : true;
  }();
  return on;
}
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Device status word at the head of the workspace (ee_get_status).
struct DevStatus {
  int32_t code;
  int32_t exit_index;
  int32_t pad[2];
};
__device__ __forceinline__ void set_status(DevStatus* st, int32_t code, int32_t exit_index) {
  if (atomicCAS(&st->code, 0, code) == 0) st->exit_index = exit_index;
}

// ---- GEMM host launcher (gemm.cu) ------------------------------------------
struct Mat {  // a row-major bf16 matrix in global memory
  const void* ptr;
  long long rows, cols, ld;  // ld in elements
};
// 2-D TMA descriptor of a bf16 matrix, SWIZZLE_128B, box [box_outer rows x box_inner cols].
bool make_tmap(CUtensorMap* m, const Mat& t, uint32_t box_inner, uint32_t box_outer);
// Operand description of one GEMM side.
//   k_major = true : storage [MN rows x K cols]  (K contiguous)
//   k_major = false: storage [K rows x MN cols]  (MN contiguous)
cudaError_t gemm_run(int epi, bool a_kmajor, bool b_kmajor, const Mat& A, const Mat& B0,
                     const Mat* B1, int b_mode, int b_ksplit, GemmArgs args, cudaStream_t st);
int num_sms();
void debug_trace_arm();
int debug_trace_read(unsigned long long* host, int max);

// ---- bandwidth-bound kernels (kernels.cu) -----------------------------------
cudaError_t launch_count_valid(const int32_t* targets, long long n, int vocab, long long* out,
                               DevStatus* st, cudaStream_t s);
// Fused all-gather target of a row-producing kernel: row t is stored into
// each of the n buffers at row row_off + t (peer pointers, include/ee.h).
constexpr int MAX_PEERS = 8;
struct PeerRows {
  __nv_bfloat16* p[MAX_PEERS];
  int n;
  long long row_off;
};
struct PeerSig {
  int* p[MAX_PEERS];
};
// rmsnorm forward; in = bf16 or fp32 [n x h] -> out bf16 [n x h], r fp32 [n]
// (ag != NULL: out is ignored and each z row goes to every ag->p[q])
cudaError_t launch_rmsnorm_fwd(const void* in, bool in_f32, const float* g, float eps,
                               __nv_bfloat16* out, float* r, long long n, int h, cudaStream_t s,
                               const PeerRows* ag = nullptr, bool pdl = false);
// rmsnorm backward: dz fp32, y (bf16/fp32), r, g -> dy bf16 (nullable), dg partials.
// dz = sum over nslots slabs dz + k*slot_stride, k = 0..nslots-1 in order
// (the fused reduce-scatter's owner-side sum).
cudaError_t launch_rmsnorm_bwd(const float* dz, const void* y, bool y_f32, const float* r,
                               const float* g, __nv_bfloat16* dy, float* dg_part, long long n,
                               int h, int rows_per_block, cudaStream_t s,
                               const __nv_bfloat16* add = nullptr,  // dy = add + dx
                               int nslots = 1, long long slot_stride = 0);
// RoPE (cos, sin) table [T x 64] for the q/k projection epilogues
cudaError_t launch_rope_table(float2* tab, int T, float theta, cudaStream_t s);
// stream-ordered barrier over peer signal arrays (int32 [MAX_PEERS] per rank)
cudaError_t launch_peer_barrier(int* const* sig, int rank, int world, unsigned epoch,
                                DevStatus* st, cudaStream_t s);
// gain grad: dg partials of sum_t du_t * x_t * r_t
cudaError_t launch_gain_grad(const float* du, const __nv_bfloat16* x, const float* r,
                             float* dg_part, long long n, int h, int rows_per_block,
                             cudaStream_t s);
cudaError_t launch_reduce_cols(const float* part, int nparts, int h, float* out, int accumulate,
                               cudaStream_t s);
cudaError_t launch_ce_finalize(const float* pm, const float* ps, const int32_t* pi,
                               const float* tl, const int32_t* targets, int nb, long long n,
                               const long long* valid_count, float alpha, float* lse, float* coef,
                               float* aux_lse, float* aux_loss, int32_t* aux_argmax,
                               float* aux_conf, float* loss_part, float* wsum_part, int nblocks,
                               cudaStream_t s);
// wsum_part != NULL: confidence weighting (L = sum w loss / sum w, written to wsum_out)
// normalize = false: L = sum w loss (the normaliser is applied by the caller later)
// a7 from the fp16 P~ the a5 epilogue stored in ds: in place -> bf16 dS
cudaError_t launch_ce_ds_from_p(__nv_bfloat16* ds, int Vl, long long n, const float* pm,
                                const float* lse, const float* coef, const int32_t* targets,
                                int vocab_begin, const float* tgt_logit, cudaStream_t s);
cudaError_t launch_loss_reduce(const float* loss_part, int nparts, const long long* valid_count,
                               const float* wsum_part, float* wsum_out, float* loss_out,
                               DevStatus* st, int exit_index, cudaStream_t s,
                               bool normalize = true);
cudaError_t launch_ce_coef_scale(float* coef, long long n, float alpha, const float* wsum,
                                 cudaStream_t s);
cudaError_t launch_scale_by_inv(float* x, long long n, const float* den, cudaStream_t s);
constexpr int FINALIZE_THREADS = 256;

// vocab-parallel softmax-CE (distributed statistics)
//   key = orderable(m) << 32 | (0xFFFFFFFF - argmax), sign-flipped so that a
//   signed int64 MAX all-reduce yields the global max and lowest-index argmax.
cudaError_t launch_vp_local_merge(const float* pm, const float* ps, const int32_t* pi,
                                  const float* tl, const int32_t* targets, int nb, long long n,
                                  int vocab_begin, int vocab_end, long long* key, float* m_loc,
                                  float* sums, cudaStream_t s);
cudaError_t launch_vp_rescale(const long long* key_global, const float* m_loc, float* sums,
                              long long n, cudaStream_t s);
cudaError_t launch_vp_finalize(const long long* key_global, const float* sums,
                               const int32_t* targets, long long n, const long long* valid_count,
                               float alpha, float* lse, float* coef, float* aux_lse,
                               float* aux_loss, int32_t* aux_argmax, float* aux_conf,
                               float* loss_part, float* wsum_part, int nblocks, cudaStream_t s);

cudaError_t launch_transpose_bf16(const __nv_bfloat16* src, __nv_bfloat16* dst, long long R, int C,
                                  long long ldd, cudaStream_t s,
                                  const float* rscale = nullptr);

cudaError_t launch_first_exit(const float* const* conf, int E, long long n, float tau,
                              int32_t* out, cudaStream_t s);

// backbone partial forward (backbone.cu)
cudaError_t launch_attn_fwd(const __nv_bfloat16* q, const __nv_bfloat16* k, const __nv_bfloat16* v,
                            __nv_bfloat16* o, long long N, int T, int Hq, int Hkv, float* lse2,
                            cudaStream_t s);
// Decode-shape exit heads (skinny.cu): M <= SKINNY_MAX_M tokens.
constexpr int SKINNY_MAX_M = 16;
enum SkinnyMode { SK_F32 = 0, SK_RESID = 1, SK_SWIGLU = 2, SK_CE = 3 };
struct SkinnyArgs {
  const __nv_bfloat16* x;  // [M x K], row stride ldx
  long long ldx;
  const __nv_bfloat16* W0;  // [N x K] row-major (SWIGLU: gate)
  const __nv_bfloat16* W1;  // SWIGLU: up
  int K, N;
  float* out;               // F32 / RESID: [M x ldo] fp32
  __nv_bfloat16* outb;      // SWIGLU: [M x ldo] bf16 = silu(x W0^T) * (x W1^T)
  long long ldo;
  const __nv_bfloat16* resid;  // RESID: [M x ldr] bf16
  long long ldr;
  float *pm, *ps;           // CE: [blocks x M] partial max / sum-exp
  int32_t* pi;              //     partial argmax (global vocab index)
  int vocab_begin;
  DevStatus* st;            // stream-K fix-up wait timeout -> EE_ERR_CUDA (or NULL)
};
cudaError_t launch_skinny(int mode, const SkinnyArgs& a, int M, cudaStream_t s);
int skinny_blocks(int N);
cudaError_t launch_infer_finalize_wide(const float* pm, const float* ps, const int32_t* pi, int nb,
                                       int M, float* lse, int32_t* argmax, float* conf,
                                       cudaStream_t s);
// tcgen05 flash-attention forward (attn_tc.cu): same contract as launch_attn_fwd,
// seq_len a multiple of 64, lse2 required.
// the two-query-tile (ping-pong) variant of the same forward
cudaError_t launch_attn_fwd_tc2(const __nv_bfloat16* q, const __nv_bfloat16* k,
                                const __nv_bfloat16* v, __nv_bfloat16* o, long long N, int T,
                                int Hq, int Hkv, float* lse2, cudaStream_t s);
cudaError_t launch_attn_fwd_tc(const __nv_bfloat16* q, const __nv_bfloat16* k,
                               const __nv_bfloat16* v, __nv_bfloat16* o, long long N, int T,
                               int Hq, int Hkv, float* lse2, cudaStream_t s);
cudaError_t launch_attn_bwd(const __nv_bfloat16* q, const __nv_bfloat16* k, const __nv_bfloat16* v,
                            const __nv_bfloat16* o, const __nv_bfloat16* dout, const float* lse2,
                            float* Dv, __nv_bfloat16* dq, __nv_bfloat16* dk, __nv_bfloat16* dv,
                            long long N, int T, int Hq, int Hkv, float rope_theta,
                            cudaStream_t s, bool tc = false,  // rope_theta > 0: fused RoPE^T
                            const float2* rope_tab = nullptr);  // (cos, sin) [T x 64] or NULL
// tcgen05 backward kernels (attn_tc.cu); Dv = rowsum(dO * O) precomputed.
cudaError_t launch_attn_bwd_tc(const __nv_bfloat16* q, const __nv_bfloat16* k,
                               const __nv_bfloat16* v, const __nv_bfloat16* dout,
                               const float* lse2, const float* Dv, __nv_bfloat16* dq,
                               __nv_bfloat16* dk, __nv_bfloat16* dv, long long N, int T, int Hq,
                               int Hkv, float rope_theta, cudaStream_t s,
                               const float2* rope_tab = nullptr);
cudaError_t launch_cast_bf16_f32(const __nv_bfloat16* a, float* b, long long n, cudaStream_t s);
cudaError_t launch_cast_f32_bf16(const float* a, __nv_bfloat16* b, long long n, cudaStream_t s);

// optimizer / init
struct OpPeers {  // every rank's operand tensor of one parameter (bf16, or fp32 if f32)
  void* p[MAX_PEERS];
  int n;
  int f32;
};
// sharded Adam: grad = rank-ordered sum of P slots [P][n]; operand rows to all ranks
cudaError_t launch_adam_sharded(float* theta, const float* slots, int P, float* m, float* v,
                                long long n, const OpPeers& op, long long off, float lr, float b1,
                                float b2, float eps, float wd, float bc1, float bc2, float gs,
                                cudaStream_t s, const float* div = nullptr);
cudaError_t launch_adam(float* theta, __nv_bfloat16* op_bf16, float* op_f32, const float* grad,
                        float* m, float* v, long long n, float lr, float b1, float b2, float eps,
                        float wd, float bc1, float bc2, float gscale, cudaStream_t s);
cudaError_t launch_sgd(float* theta, __nv_bfloat16* op_bf16, float* op_f32, const float* grad,
                       float* buf, long long n, float lr, float mom, float gscale, cudaStream_t s);
cudaError_t launch_copy_cast(const void* src, bool src_f32, float* master, __nv_bfloat16* op_bf16,
                             float* op_f32, long long n, cudaStream_t s);
cudaError_t launch_random_normal(uint64_t seed, uint64_t stream_id, float std, float* master,
                                 __nv_bfloat16* op_bf16, long long n, cudaStream_t s);
cudaError_t launch_fill(float* master, float* op_f32, long long n, float value, cudaStream_t s);

}  // namespace ee
