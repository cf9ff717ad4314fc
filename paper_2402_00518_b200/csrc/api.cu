// api.cu -- the C-ABI (include/ee.h): argument validation, workspace carving
// and the per-exit kernel sequence of one EE-Tuning step.
//
// Per exit i, all on `stream`:
//   MLP only   a1  u = RMSNorm_a(x)                      rmsnorm_fwd        (HBM)
//              a2  [A|B] = u [W_gate|W_up]^T, M = silu(A)B  GEMM+SwiGLU    (tensor)
//              a3  y = x + M W_down^T                    GEMM+residual      (tensor)
//   Norm/MLP   a4  z = RMSNorm_f(y)                      rmsnorm_fwd        (HBM)
//   all        a5  per-tile online-softmax stats of z W_out^T  GEMM+CE     (tensor)
//              a6  lse, loss_t, argmax, conf, L_i        ce_finalize/reduce (HBM)
//              a7  dS = coef (softmax - onehot), recomputed GEMM -> bf16    (tensor)
//   Norm/MLP   a8  dz = dS W_out                         GEMM (B MN-major)  (tensor)
//   all        a9  dW_out = dS^T z                       GEMM (A,B MN-major)(tensor)
//   Norm/MLP   a10 dg_f, dy                              rmsnorm_bwd        (HBM)
//   MLP only   a11 dW_down = dy^T M; dM = dy W_down -> dA, dB (SwiGLU bwd epilogue)
//              a12 dW_gate|up = [dA|dB]^T u; du = [dA|dB] [W_gate;W_up]
//              a13 dg_a = sum du * xhat                  gain_grad          (HBM)
// The full [tokens x vocab] logit matrix is never written: a5 keeps only
// per-tile (max, sum-exp, argmax) partials and a7 recomputes S tile by tile.
#include <cuda.h>
#include <cuda_runtime.h>
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdarg>
#include <cstring>
#include <string>
#include <atomic>
#include <vector>
#include <nvtx3/nvToolsExt.h>
#include "../../include/ee.h"
#include "internal.cuh"

using namespace ee;

namespace ee {
// NVTX range on the calling host thread (per exit and per phase of the step;
// a no-op unless a profiler such as nsys is attached).
struct Nvtx {
  explicit Nvtx(const char* fmt, int i = -1) {
    char b[96];
    if (i >= 0) snprintf(b, sizeof(b), fmt, i); else snprintf(b, sizeof(b), "%s", fmt);
    nvtxRangePushA(b);
  }
  ~Nvtx() { nvtxRangePop(); }
};
}  // namespace ee

namespace {

thread_local std::string g_last_error;

ee_status fail(ee_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return s;
}

#define EE_CUDA(call)                                                                         \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      return fail(EE_ERR_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_),        \
                  __FILE__, __LINE__);                                                        \
  } while (0)

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

constexpr int NORM_RPB = 64;  // rows per block of the norm backward / gain-grad kernels

ee_status check_cfg(const ee_head_config* c) {
  if (!c) return fail(EE_ERR_ARG, "cfg is NULL");
  if (c->arch < EE_ARCH_EMBEDDING || c->arch > EE_ARCH_LAYER)
    return fail(EE_ERR_ARG, "unknown arch %d", c->arch);
  if (c->num_exits < 1) return fail(EE_ERR_ARG, "num_exits must be >= 1");
  if (c->hidden < 64 || c->hidden > 8192 || c->hidden % 64 != 0)
    return fail(EE_ERR_SHAPE, "hidden must be a multiple of 64 in [64, 8192], got %d", c->hidden);
  if (c->vocab < 1) return fail(EE_ERR_SHAPE, "vocab must be >= 1");
  if (c->vocab_begin < 0 || c->vocab_end > c->vocab || c->vocab_begin >= c->vocab_end)
    return fail(EE_ERR_SHAPE, "vocab shard [%d, %d) outside [0, %d)", c->vocab_begin, c->vocab_end,
                c->vocab);
  if ((c->vocab_end - c->vocab_begin) % 8 != 0)
    return fail(EE_ERR_SHAPE, "local vocab size must be a multiple of 8");
  if (c->arch >= EE_ARCH_MLP && (c->ffn < 128 || c->ffn % 128 != 0))
    return fail(EE_ERR_SHAPE, "ffn must be a positive multiple of 128 for MLP/Layer exits, got %d",
                c->ffn);
  if (c->arch == EE_ARCH_LAYER) {
    if (c->n_heads < 1 || c->n_kv_heads < 1 || c->n_heads % c->n_kv_heads != 0)
      return fail(EE_ERR_SHAPE, "Layer exit: n_kv_heads must divide n_heads (%d, %d)", c->n_heads,
                  c->n_kv_heads);
    if (c->hidden != 128 * c->n_heads)
      return fail(EE_ERR_SHAPE, "Layer exit: hidden must be n_heads * 128 (head dim 128)");
    if (c->seq_len < 64 || c->seq_len % 64 != 0)
      return fail(EE_ERR_SHAPE, "Layer exit: seq_len must be a positive multiple of 64");
    if (!(c->rope_theta > 0.f)) return fail(EE_ERR_ARG, "Layer exit: rope_theta must be > 0");
  }
  if (!(c->norm_eps >= 0.f)) return fail(EE_ERR_ARG, "norm_eps must be >= 0");
  if (c->token_weighting != EE_WEIGHT_UNIFORM && c->token_weighting != EE_WEIGHT_CONFIDENCE &&
      c->token_weighting != EE_WEIGHT_CONFIDENCE_SUM)
    return fail(EE_ERR_ARG, "unknown token_weighting %d", c->token_weighting);
  if (c->ds_mode != EE_DS_RECOMPUTE && c->ds_mode != EE_DS_STORED_P)
    return fail(EE_ERR_ARG, "unknown ds_mode %d", c->ds_mode);
  return EE_OK;
}

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

// Layer exits couple the tokens of a sequence: a call must hold whole sequences.
ee_status check_tokens(const ee_head_config* c, long long n) {
  if (c->arch == EE_ARCH_LAYER && n % c->seq_len != 0)
    return fail(EE_ERR_SHAPE, "Layer exit: n_tokens (%lld) must be a multiple of seq_len (%d)", n,
                c->seq_len);
  return EE_OK;
}

// The exit tensors in ee_head_tensors order; Random-init streams are keyed by
// this index (exit * 16 + k).
constexpr int NTENS = 11;
struct TInfo {
  void* ee_head_tensors::*f;
  const char* name;
  bool gain, vocab;
};
const TInfo kTens[NTENS] = {
    {&ee_head_tensors::g_a, "g_a", true, false},       {&ee_head_tensors::w_gate, "w_gate", false, false},
    {&ee_head_tensors::w_up, "w_up", false, false},    {&ee_head_tensors::w_down, "w_down", false, false},
    {&ee_head_tensors::g_f, "g_f", true, false},       {&ee_head_tensors::w_out, "w_out", false, true},
    {&ee_head_tensors::g_att, "g_att", true, false},   {&ee_head_tensors::w_q, "w_q", false, false},
    {&ee_head_tensors::w_k, "w_k", false, false},      {&ee_head_tensors::w_v, "w_v", false, false},
    {&ee_head_tensors::w_o, "w_o", false, false}};

// Row geometry of tensor k as a [R x C] matrix (gains: one row) and its
// row-block sharding over P ranks for the fused data-parallel path (ZeRO-1):
// chunk = ceil(R / P) rows per owner, owner q holds rows [q*chunk, ...).
void tensor_rc(const ee_head_config* c, int k, long long* R, long long* C) {
  const long long h = c->hidden, F = c->ffn, Vl = c->vocab_end - c->vocab_begin;
  const long long hkv = 128LL * c->n_kv_heads;
  switch (k) {
    case 0: case 4: case 6: *R = 1; *C = h; return;
    case 1: case 2: *R = F; *C = h; return;
    case 3: *R = h; *C = F; return;
    case 5: *R = Vl; *C = h; return;
    case 7: case 10: *R = h; *C = h; return;
    default: *R = hkv; *C = h; return;
  }
}
long long shard_chunk(long long R, int P) { return (R + P - 1) / P; }
long long shard_rows(long long R, int P, int q) {
  const long long ch = shard_chunk(R, P), b = q * ch;
  return b >= R ? 0 : (R - b < ch ? R - b : ch);
}
bool tensor_needed(const ee_head_config* c, int k);
// float offset of tensor k's slot block [P][rows_q x C] in rank q's arena; k = NTENS: total
// Under a vocab shard (vocab-parallel) W_out is never reduced and its row count
// differs between ranks, so it has no arena block: every rank must compute the
// same offsets for every owner.
static bool in_arena(const ee_head_config* c, int k) {
  if (!tensor_needed(c, k)) return false;
  return !(k == 5 && (c->vocab_begin != 0 || c->vocab_end != c->vocab));
}
long long arena_offset(const ee_head_config* c, int P, int q, int k) {
  long long off = 0;
  for (int j = 0; j < k; ++j) {
    if (!in_arena(c, j)) continue;
    long long R, C;
    tensor_rc(c, j, &R, &C);
    off += (long long)P * shard_rows(R, P, q) * C;
  }
  return off;
}

bool tensor_needed(const ee_head_config* c, int k) {
  if (k == 5) return true;                          // w_out
  if (k == 4) return c->arch != EE_ARCH_EMBEDDING;  // g_f
  if (k < 4) return c->arch >= EE_ARCH_MLP;         // MLP body
  return c->arch == EE_ARCH_LAYER;                  // attention block
}

long long tensor_numel(const ee_head_config* c, int k) {
  const long long h = c->hidden, F = c->ffn, Vl = c->vocab_end - c->vocab_begin;
  const long long hkv = 128LL * c->n_kv_heads;
  switch (k) {
    case 0: case 4: case 6: return h;
    case 1: case 2: case 3: return F * h;
    case 5: return Vl * h;
    case 7: case 10: return h * h;
    default: return hkv * h;  // w_k, w_v
  }
}

struct Layout {
  size_t wsum_part, wsum, zT, uT, dyT, gsc;
  long long ldT;  // leading dimension of the transposed [h x n] copies (n rounded up to 8)
  size_t status, vcount, loss_part, lse, coef, tgt, pm, ps, pi, z, ds, dz, dgp, ry, u, rx, ab,
      mact, y, dy, total;
  // Layer exits: attention block activations / gradients
  size_t u1, r1, q, k, v, o, lse2, x1, da, dq, dk, dv, dvec, rope;
  int nb, nparts, nfin;
};

Layout make_layout(const ee_head_config* c, long long n) {
  Layout L{};
  const long long h = c->hidden, Vl = c->vocab_end - c->vocab_begin, F = c->ffn;
  L.nb = (int)((Vl + GEMM_BN - 1) / GEMM_BN);
  L.nparts = (int)((n + NORM_RPB - 1) / NORM_RPB);
  L.nfin = (int)((n + FINALIZE_THREADS - 1) / FINALIZE_THREADS);
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t r = o;
    o = align_up(o + bytes);
    return r;
  };
  L.status = take(sizeof(DevStatus));
  L.gsc = take(4 * 3 * (size_t)h);  // fused Adam: g_f / g_a / g_att gradients
  L.vcount = take(8);
  L.loss_part = take(4 * (size_t)(L.nfin > 0 ? L.nfin : 1));
  L.wsum_part = take(4 * (size_t)(L.nfin > 0 ? L.nfin : 1));
  L.wsum = take(4);
  L.lse = take(4 * n);
  L.coef = take(4 * n);
  L.tgt = take(4 * n);
  L.pm = take(4 * (size_t)L.nb * n);
  L.ps = take(4 * (size_t)L.nb * n);
  L.pi = take(4 * (size_t)L.nb * n);
  L.ds = take(2 * (size_t)n * Vl);
  L.ldT = (n + 7) / 8 * 8;
  L.zT = take(2 * (size_t)h * L.ldT);
  L.uT = L.dyT = 0;
  L.z = L.dz = L.dgp = L.ry = L.u = L.rx = L.ab = L.mact = L.y = L.dy = 0;
  if (c->arch != EE_ARCH_EMBEDDING) {
    L.z = take(2 * (size_t)n * h);
    L.dz = take(4 * (size_t)n * h);
    // column-sum partials: RMSNorm row blocks, or (MLP exits) dW-GEMM column blocks
    size_t gp = (size_t)(L.nparts > 0 ? L.nparts : 1);
    if (c->arch == EE_ARCH_MLP && n > 0) gp = std::max(gp, (size_t)((2 * F + GEMM_BN - 1) / GEMM_BN));
    L.dgp = take(4 * gp * h);
    L.ry = take(4 * n);
  }
  L.u1 = L.r1 = L.q = L.k = L.v = L.o = L.lse2 = L.x1 = L.da = L.dq = L.dk = L.dv = L.dvec = 0;
  if (c->arch >= EE_ARCH_MLP) {
    L.u = take(2 * (size_t)n * h);
    L.rx = take(4 * n);
    L.ab = take(2 * (size_t)n * 2 * F);
    L.mact = take(2 * (size_t)n * F);
    L.y = take(4 * (size_t)n * h);
    L.dy = take(2 * (size_t)n * h);
    L.uT = take(2 * (size_t)h * L.ldT);
    L.dyT = take(2 * (size_t)h * L.ldT);
  }
  if (c->arch == EE_ARCH_LAYER) {
    const long long hkv = 128LL * c->n_kv_heads, Hq = c->n_heads;
    L.u1 = take(2 * (size_t)n * h);
    L.r1 = take(4 * n);
    L.q = take(2 * (size_t)n * h);
    L.k = take(2 * (size_t)n * hkv);
    L.v = take(2 * (size_t)n * hkv);
    L.o = take(2 * (size_t)n * h);
    L.lse2 = take(4 * (size_t)n * Hq);
    L.x1 = take(4 * (size_t)n * h);
    L.da = take(2 * (size_t)n * h);
    L.dq = take(2 * (size_t)n * h);
    L.dk = take(2 * (size_t)n * hkv);
    L.dv = take(2 * (size_t)n * hkv);
    L.dvec = take(4 * (size_t)n * Hq);
    L.rope = take(8 * 64 * (size_t)c->seq_len);
  }
  L.total = o;
  return L;
}

ee_status check_device() {
  static int ok = -1;
  if (ok < 0) {
    int dev = 0;
    cudaDeviceProp p;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaGetDeviceProperties(&p, dev) != cudaSuccess) {
      cudaGetLastError();
      ok = 0;
    } else {
      ok = (p.major == 10 && p.minor == 0) ? 1 : 0;
    }
  }
  if (!ok) return fail(EE_ERR_UNSUPPORTED, "no sm_100 (B200) device is current");
  return EE_OK;
}

ee_status check_arch_tensors(const ee_head_config* c, const ee_head_tensors& t, const char* what,
                             int i) {
  for (int k = 0; k < NTENS; ++k) {
    const void* p = t.*(kTens[k].f);
    if (tensor_needed(c, k) != (p != nullptr))
      return fail(EE_ERR_ARCH, "%s[%d].%s is %s for arch %d", what, i, kTens[k].name,
                  p ? "set but unused" : "NULL but required", c->arch);
    if (p && !aligned16(p)) return fail(EE_ERR_ALIGN, "%s[%d].%s not 16-byte aligned", what, i,
                                        kTens[k].name);
  }
  return EE_OK;
}


// ---------------------------------------------------------------- profiler
// Optional per-launch CUDA-event timing (ee_profile_*): one event pair per
// kernel launch, recorded on the launching stream, so bench.py can report the
// duration and algorithmic FLOPs / bytes of each kernel inside its timed region.
struct ProfRec {
  const char* name;
  cudaEvent_t a, b;
  double flops_exec, flops_alg, bytes;
};
std::vector<ProfRec> g_prof;
std::vector<cudaEvent_t> g_event_pool;
bool g_prof_on = false;
std::atomic<long long> g_launches{0};

cudaEvent_t pool_event() {
  if (!g_event_pool.empty()) {
    cudaEvent_t e = g_event_pool.back();
    g_event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

struct Prof {
  bool on;
  size_t idx;
  cudaStream_t st;
  Prof(const char* name, cudaStream_t s, double fe, double fa, double by) : on(g_prof_on), st(s) {
    ++g_launches;
    if (!on) return;
    ProfRec r{name, pool_event(), pool_event(), fe, fa, by};
    cudaEventRecord(r.a, st);
    idx = g_prof.size();
    g_prof.push_back(r);
  }
  ~Prof() {
    if (on) cudaEventRecord(g_prof[idx].b, st);
  }
};

// Attention kernels (attn_tc.cu): EE_ATTN_TC = 2 (default) the two-query-tile
// tcgen05 forward, 1 the one-tile tcgen05 forward, 0 the mma.sync kernels
// (A/B measurements; the backward is tcgen05 unless 0).
int attn_tc_mode() {
  static const int tc = [] {
    const char* e = getenv("EE_ATTN_TC");
    return e ? atoi(e) : 2;
  }();
  return tc;
}
cudaError_t attn_forward_impl(int impl, const __nv_bfloat16* q, const __nv_bfloat16* k,
                              const __nv_bfloat16* v, __nv_bfloat16* o, long long n, int T,
                              int Hq, int Hkv, float* lse2, cudaStream_t st) {
  if (impl == 2) return launch_attn_fwd_tc2(q, k, v, o, n, T, Hq, Hkv, lse2, st);
  if (impl == 1) return launch_attn_fwd_tc(q, k, v, o, n, T, Hq, Hkv, lse2, st);
  return launch_attn_fwd(q, k, v, o, n, T, Hq, Hkv, lse2, st);
}
cudaError_t attn_forward(const __nv_bfloat16* q, const __nv_bfloat16* k, const __nv_bfloat16* v,
                         __nv_bfloat16* o, long long n, int T, int Hq, int Hkv, float* lse2,
                         cudaStream_t st) {
  return attn_forward_impl(attn_tc_mode(), q, k, v, o, n, T, Hq, Hkv, lse2, st);
}

GemmArgs base_args(int M, int N, int K) {
  GemmArgs a;
  memset(&a, 0, sizeof(a));
  a.M = M;
  a.N = N;
  a.K = K;
  a.m_split = M;
  a.n_split = N;
  a.group_m = 16;
  return a;
}

}  // namespace

namespace ee {
ee_status comm_fail(ee_status s, const char* msg) { return fail(s, "%s", msg); }
ee_status comm_tune_step(const ee_comm* c, const ee_head_config* cfg, const void* const* hidden,
                         int64_t n_tokens, const int32_t* targets, const float* exit_weights,
                         const ee_head_tensors* params, ee_head_tensors* grads, int32_t accumulate,
                         float* loss_out, const ee_step_aux* aux, const int64_t* valid_count,
                         void* workspace, size_t ws_bytes, void* stream);   // comm.cu
}  // namespace ee

extern "C" {

const char* ee_last_error(void) { return g_last_error.c_str(); }
const char* ee_version(void) { return "ee_b200 0.1.0 (sm_100a tcgen05)"; }

double ee_lr_at(int64_t it, int64_t total, double warmup_frac, double lr_max, double lr_min) {
  if (total < 1 || it < 0 || it > total) return NAN;
  const int64_t w = (int64_t)std::ceil(warmup_frac * (double)total);
  if (w > 0 && it <= w) return lr_max * (double)it / (double)w;
  if (total == w) return lr_max;
  return lr_max - (lr_max - lr_min) * (double)(it - w) / (double)(total - w);
}

ee_status ee_workspace_size(const ee_head_config* cfg, int64_t n_tokens, size_t* bytes) {
  ee_status s = check_cfg(cfg);
  if (s != EE_OK) return s;
  if (!bytes || n_tokens < 0) return fail(EE_ERR_ARG, "bytes NULL or n_tokens < 0");
  *bytes = make_layout(cfg, n_tokens).total;
  return EE_OK;
}

ee_status ee_get_status(void* workspace, void* stream, int32_t* code, int32_t* exit_index) {
  if (!workspace || !code || !exit_index) return fail(EE_ERR_ARG, "NULL argument");
  cudaStream_t st = (cudaStream_t)stream;
  DevStatus h{};
  EE_CUDA(cudaMemcpyAsync(&h, workspace, sizeof(h), cudaMemcpyDeviceToHost, st));
  EE_CUDA(cudaStreamSynchronize(st));
  *code = h.code;
  *exit_index = h.code ? h.exit_index : -1;
  if (h.code) {
    EE_CUDA(cudaMemsetAsync(workspace, 0, sizeof(DevStatus), st));
    EE_CUDA(cudaStreamSynchronize(st));
  }
  return EE_OK;
}

ee_status ee_count_valid(const int32_t* targets, int64_t n, int32_t vocab, int64_t* out,
                         void* workspace, size_t ws_bytes, void* stream) {
  if (!out || !workspace || (n > 0 && !targets)) return fail(EE_ERR_ARG, "NULL argument");
  if (ws_bytes < sizeof(DevStatus)) return fail(EE_ERR_WORKSPACE, "workspace too small");
  ee_status s = check_device();
  if (s != EE_OK) return s;
  EE_CUDA(launch_count_valid(targets, n, vocab, (long long*)out, (DevStatus*)workspace,
                             (cudaStream_t)stream));
  return EE_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- step phases
namespace {

// Workspace views for one call (layout sized for n tokens).
struct Bufs {
  DevStatus* status;
  long long* vcount;
  float *lse, *coef, *tgt, *pm, *ps, *loss_part, *wsum_part, *wsum;
  int32_t* pi;
  __nv_bfloat16* ds;
  __nv_bfloat16* z;
  float *dz, *dgp, *ry;
  __nv_bfloat16* u;
  float* rx;
  __nv_bfloat16 *ab, *mact;
  float* y;
  __nv_bfloat16* dy;
  __nv_bfloat16 *zT, *uT, *dyT;  // K-major copies for the weight-gradient GEMMs
  // Layer exits
  __nv_bfloat16 *u1, *q, *k, *v, *o, *da, *dq, *dk, *dv;
  float *r1, *lse2, *x1, *dvec;
  float2* rope;
  // vocab-parallel merge state
  float* m_loc;
  float* gsc;  // [2 x h] gain gradients of ee_tune_step_adam
  Layout L;
};

Bufs make_bufs(const ee_head_config* cfg, long long n, void* workspace) {
  Bufs B{};
  B.L = make_layout(cfg, n);
  const Layout& L = B.L;
  uint8_t* ws = (uint8_t*)workspace;
  const bool mlp = cfg->arch >= EE_ARCH_MLP, nrm = cfg->arch != EE_ARCH_EMBEDDING;
  B.status = (DevStatus*)(ws + L.status);
  B.gsc = (float*)(ws + L.gsc);
  B.vcount = (long long*)(ws + L.vcount);
  B.lse = (float*)(ws + L.lse);
  B.coef = (float*)(ws + L.coef);
  B.tgt = (float*)(ws + L.tgt);
  B.pm = (float*)(ws + L.pm);
  B.ps = (float*)(ws + L.ps);
  B.pi = (int32_t*)(ws + L.pi);
  B.loss_part = (float*)(ws + L.loss_part);
  B.wsum_part = (float*)(ws + L.wsum_part);
  B.wsum = (float*)(ws + L.wsum);
  B.ds = (__nv_bfloat16*)(ws + L.ds);
  B.m_loc = B.coef;  // VP: m_loc is dead before coef is written (vp_finalize)
  B.zT = (__nv_bfloat16*)(ws + L.zT);
  if (nrm) {
    B.z = (__nv_bfloat16*)(ws + L.z);
    B.dz = (float*)(ws + L.dz);
    B.dgp = (float*)(ws + L.dgp);
    B.ry = (float*)(ws + L.ry);
  }
  if (mlp) {
    B.u = (__nv_bfloat16*)(ws + L.u);
    B.rx = (float*)(ws + L.rx);
    B.ab = (__nv_bfloat16*)(ws + L.ab);
    B.mact = (__nv_bfloat16*)(ws + L.mact);
    B.y = (float*)(ws + L.y);
    B.dy = (__nv_bfloat16*)(ws + L.dy);
    B.uT = (__nv_bfloat16*)(ws + L.uT);
    B.dyT = (__nv_bfloat16*)(ws + L.dyT);
  }
  if (cfg->arch == EE_ARCH_LAYER) {
    B.u1 = (__nv_bfloat16*)(ws + L.u1);
    B.r1 = (float*)(ws + L.r1);
    B.q = (__nv_bfloat16*)(ws + L.q);
    B.k = (__nv_bfloat16*)(ws + L.k);
    B.v = (__nv_bfloat16*)(ws + L.v);
    B.o = (__nv_bfloat16*)(ws + L.o);
    B.lse2 = (float*)(ws + L.lse2);
    B.x1 = (float*)(ws + L.x1);
    B.da = (__nv_bfloat16*)(ws + L.da);
    B.dq = (__nv_bfloat16*)(ws + L.dq);
    B.dk = (__nv_bfloat16*)(ws + L.dk);
    B.dv = (__nv_bfloat16*)(ws + L.dv);
    B.dvec = (float*)(ws + L.dvec);
    B.rope = (float2*)(ws + L.rope);
  }
  return B;
}

// ---- Layer exit, attention block (Llama-2 layer P:356-358) ----
// L1 u1 = RMSNorm_att(x); L2 q|k|v = u1 W^T with L3 RoPE(q, k) fused into the
// projection epilogues; L4 causal GQA flash
// attention (o, lse2); L5 x1 = x + o W_o^T (fp32 residual stream, A15).
ee_status layer_attn_forward(const ee_head_config* cfg, const Bufs& B, const ee_head_tensors& P,
                             const __nv_bfloat16* x, long long n, cudaStream_t st) {
  const int h = cfg->hidden, Hq = cfg->n_heads, Hkv = cfg->n_kv_heads, hkv = 128 * Hkv;
  { Prof p_("L1_rmsnorm_att", st, 0, 0, 4.0 * n * h + 4.0 * n);
  EE_CUDA(launch_rmsnorm_fwd(x, false, (const float*)P.g_att, cfg->norm_eps, B.u1, B.r1, n, h, st)); }
  struct Proj {
    const void* w;
    __nv_bfloat16* out;
    int N;
    const char* name;
  } projs[3] = {{P.w_q, B.q, h, "L2_q_proj"}, {P.w_k, B.k, hkv, "L2_k_proj"},
                {P.w_v, B.v, hkv, "L2_v_proj"}};
  EE_CUDA(launch_rope_table(B.rope, cfg->seq_len, cfg->rope_theta, st));
  for (int j = 0; j < 3; ++j) {  // L3: RoPE fused into the q / k epilogues (fp32, one rounding)
    const Proj& pj = projs[j];
    GemmArgs a = base_args((int)n, pj.N, h);
    a.outb = pj.out;
    a.ldo = pj.N;
    if (j < 2) {
      a.rope_seq = cfg->seq_len;
      a.rope_theta = cfg->rope_theta;
      a.rope_tab = B.rope;
    }
    Mat A{B.u1, n, h, h}, Bm{pj.w, pj.N, h, h};
    Prof p_(pj.name, st, 2.0 * n * pj.N * h, 2.0 * n * pj.N * h, 0);
    EE_CUDA(gemm_run(EPI_BF16, true, true, A, Bm, nullptr, B_PLAIN, 0, a, st));
  }
  { const double fl = 2.0 * (double)n * h * (cfg->seq_len + 1);  // causal: 2 GEMMs x T/2 keys
    Prof p_("L4_attn_fwd", st, 2.0 * (double)n * h * (cfg->seq_len + 64), fl, 0);
    EE_CUDA(attn_forward(B.q, B.k, B.v, B.o, n, cfg->seq_len, Hq, Hkv, B.lse2, st)); }
  {
    GemmArgs a = base_args((int)n, h, h);
    a.out0 = B.x1;
    a.ldo = h;
    a.resid = x;
    a.ld_resid = h;
    Mat A{B.o, n, h, h}, Bm{P.w_o, h, h, h};
    Prof p_("L5_o_proj_resid", st, 2.0 * n * h * h, 2.0 * n * h * h, 0);
    EE_CUDA(gemm_run(EPI_RESID, true, true, A, Bm, nullptr, B_PLAIN, 0, a, st));
  }
  return EE_OK;
}

// Backward of the attention block given dx1 (bf16, in B.dy): L6 dW_o = dx1^T o;
// L7 da = dx1 W_o; L8 flash-attention backward (dq, dk, dv) with L9 RoPE^T
// fused into its dq / dk stores;
// L10 dW_{q,k,v} = d{q,k,v}^T u1; L11 du1 = dq W_q + dk W_k + dv W_v;
// L12 dg_att = sum du1 * xhat1 (no dx: frozen backbone).
struct GradScatter;
static void set_scatter(GemmArgs& a, const GradScatter* gs, int k, int k1);
static float* scatter_gain(const GradScatter* gs, int k);
struct AdamFuse;
static void set_adam(GemmArgs& a, const AdamFuse* af, int k, int k1);

ee_status layer_attn_backward(const ee_head_config* cfg, const Bufs& B, const ee_head_tensors& P,
                              const ee_head_tensors& G, const __nv_bfloat16* x, long long n,
                              int accumulate, cudaStream_t st, const GradScatter* gs = nullptr,
                              const AdamFuse* af = nullptr, float* gain_grad = nullptr) {
  const int h = cfg->hidden, Hq = cfg->n_heads, Hkv = cfg->n_kv_heads, hkv = 128 * Hkv;
  const int nparts = (int)((n + NORM_RPB - 1) / NORM_RPB);
  {  // L7: da = dx1 W_o  (W_o read MN-major in place; before L6, which may update W_o)
    GemmArgs a = base_args((int)n, h, h);
    a.outb = B.da;
    a.ldo = h;
    Mat A{B.dy, n, h, h}, Bm{P.w_o, h, h, h};
    Prof p_("L7_da", st, 2.0 * n * h * h, 2.0 * n * h * h, 0);
    EE_CUDA(gemm_run(EPI_BF16, true, false, A, Bm, nullptr, B_PLAIN, 0, a, st));
  }
  {  // L6: dW_o = dx1^T o  (A = dx1^T K-major copy, B = o MN-major)
    { Prof p_("transpose_dx1", st, 0, 0, 4.0 * n * h);
    EE_CUDA(launch_transpose_bf16(B.dy, B.dyT, n, h, B.L.ldT, st)); }
    GemmArgs a = base_args(h, h, (int)n);
    a.out0 = (float*)G.w_o;
    a.ldo = h;
    a.accumulate = accumulate;
    if (gs) set_scatter(a, gs, 10, -1);
    if (af) set_adam(a, af, 10, -1);
    Mat A{B.dyT, h, n, B.L.ldT}, Bm{B.o, n, h, h};
    Prof p_("L6_dw_o", st, 2.0 * n * h * h, 2.0 * n * h * h, 0);
    EE_CUDA(gemm_run(af ? EPI_F32_ADAM : EPI_F32, true, false, A, Bm, nullptr, B_PLAIN, 0, a,
                     st));
  }
  { const double fa = 4.0 * (double)n * h * (cfg->seq_len + 1);    // dV, dP, dQ, dK
    const double fe = 7.0 * (double)n * h * (cfg->seq_len + 64);   // + S twice, dP twice
    Prof p_("L8_attn_bwd", st, fe, fa, 0);
    EE_CUDA(launch_attn_bwd(B.q, B.k, B.v, B.o, B.da, B.lse2, B.dvec, B.dq, B.dk, B.dv, n,
                            cfg->seq_len, Hq, Hkv, cfg->rope_theta, st,
                            attn_tc_mode() != 0, B.rope)); }  // + L9 RoPE^T fused
  { Prof p_("transpose_u1", st, 0, 0, 4.0 * n * h);
  EE_CUDA(launch_transpose_bf16(B.u1, B.uT, n, h, B.L.ldT, st)); }
  struct WG {
    const __nv_bfloat16* d;
    void* g;
    const void* w;
    int N;
    const char *name, *dname;
    int k;  // tensor index (ee_head_tensors order)
  } wg[3] = {{B.dq, G.w_q, P.w_q, h, "L10_dw_q", "L11_du1_q", 7},
             {B.dk, G.w_k, P.w_k, hkv, "L10_dw_k", "L11_du1_k", 8},
             {B.dv, G.w_v, P.w_v, hkv, "L10_dw_v", "L11_du1_v", 9}};
  for (int j = 0; j < 3; ++j) {  // L11: du1 (+)= d W  (W read MN-major in place) -> B.dz
    const WG& w = wg[j];
    GemmArgs a = base_args((int)n, h, w.N);
    a.out0 = B.dz;
    a.ldo = h;
    a.accumulate = j > 0;
    Mat A{w.d, n, w.N, w.N}, Bm{w.w, w.N, h, h};
    Prof p_(w.dname, st, 2.0 * n * w.N * h, 2.0 * n * w.N * h, 0);
    EE_CUDA(gemm_run(EPI_F32, true, false, A, Bm, nullptr, B_PLAIN, 0, a, st));
  }
  for (const WG& w : wg) {  // L10 (after L11, which reads W_q/k/v): dW^T = u1^T d (A = u1^T K-major, B = d MN-major), stored transposed
    GemmArgs a = base_args(h, w.N, (int)n);
    a.out0 = (float*)w.g;
    a.ldo = h;
    a.n_split = w.N;
    a.accumulate = accumulate;
    if (gs) set_scatter(a, gs, w.k, -1);
    if (af) set_adam(a, af, w.k, -1);
    Mat A{B.uT, h, n, B.L.ldT}, Bm{w.d, n, w.N, w.N};
    Prof p_(w.name, st, 2.0 * n * w.N * h, 2.0 * n * w.N * h, 0);
    EE_CUDA(gemm_run(af ? EPI_F32T_ADAM : EPI_F32T, true, false, A, Bm, nullptr, B_PLAIN, 0, a,
                     st));
  }
  { Prof p_("L12_gain_grad", st, 0, 0, 6.0 * n * h);
  EE_CUDA(launch_gain_grad(B.dz, x, B.r1, B.dgp, n, h, NORM_RPB, st)); }
  { Prof p_("reduce_cols", st, 0, 0, 4.0 * nparts * h);
  EE_CUDA(launch_reduce_cols(B.dgp, nparts, h,
                             gs ? scatter_gain(gs, 6) : af ? gain_grad : (float*)G.g_att,
                             accumulate, st)); }
  return EE_OK;
}

// Fused Adam (ee_tune_step_adam): per tensor k the state the weight-gradient
// epilogue updates in place instead of storing the gradient.
struct AdamFuse {
  AdamOut t[NTENS];
  AdamScal sc;
};

static void set_adam(GemmArgs& a, const AdamFuse* af, int k, int k1) {
  a.adam_on = 1;
  a.adam = af->sc;
  a.adam0 = af->t[k];
  if (k1 >= 0) a.adam1 = af->t[k1];
}

// Fused data-parallel gradient routing (ee_tune_step_rs): p[k][q] = where
// this rank's partial of tensor k's rows owned by rank q go (owner q's arena,
// slot [rank]); chunk[k] = rows per owner.  Gains: one row, owner 0.
struct GradScatter {
  float* p[NTENS][MAX_PEERS];
  int chunk[NTENS];
};

static GradScatter make_scatter(const ee_head_config* c, const ee_peer_set& arenas) {
  GradScatter g;
  memset(&g, 0, sizeof(g));
  const int P = arenas.world;
  for (int k = 0; k < NTENS; ++k) {
    if (!in_arena(c, k)) continue;
    long long R, C;
    tensor_rc(c, k, &R, &C);
    g.chunk[k] = (int)shard_chunk(R, P);
    for (int q = 0; q < P; ++q)
      g.p[k][q] = (float*)arenas.ptr[q] + arena_offset(c, P, q, k) +
                  (long long)arenas.rank * shard_rows(R, P, q) * C;
  }
  return g;
}

static float* scatter_gain(const GradScatter* gs, int k) { return gs->p[k][0]; }

static void set_scatter(GemmArgs& a, const GradScatter* gs, int k, int k1) {
  a.scat_rows = gs->chunk[k];
  for (int q = 0; q < MAX_PEERS; ++q) {
    a.scat[q] = gs->p[k][q];
    a.scat1[q] = k1 >= 0 ? gs->p[k1][q] : nullptr;
  }
}

// a1..a4: z = exit-head input of the vocab projection, on n tokens.
// z_out: where to write z (NULL = the workspace buffer; Embedding: z = x unless
// z_out is given, in which case x is copied there).  Returns z in *z_ret.
ee_status phase_exit_forward(const ee_head_config* cfg, const Bufs& B, const ee_head_tensors& P,
                             const __nv_bfloat16* x, long long n, __nv_bfloat16* z_out,
                             const __nv_bfloat16** z_ret, cudaStream_t st,
                             const PeerRows* ag = nullptr) {
  const int h = cfg->hidden, F = cfg->ffn;
  const bool mlp = cfg->arch >= EE_ARCH_MLP, nrm = cfg->arch != EE_ARCH_EMBEDDING;
  const bool layer = cfg->arch == EE_ARCH_LAYER;
  if (!nrm) {
    if (ag) {  // fused all-gather of z = x: one copy into every rank's z_all
      for (int q = 0; q < ag->n && n > 0; ++q)
        EE_CUDA(cudaMemcpyAsync(ag->p[q] + ag->row_off * h, x, 2 * (size_t)n * h,
                                cudaMemcpyDefault, st));
      *z_ret = nullptr;
      return EE_OK;
    }
    if (z_out && n > 0)
      EE_CUDA(cudaMemcpyAsync(z_out, x, 2 * (size_t)n * h, cudaMemcpyDeviceToDevice, st));
    *z_ret = z_out ? z_out : x;
    return EE_OK;
  }
  __nv_bfloat16* z = z_out ? z_out : B.z;
  *z_ret = z;
  if (n == 0) return EE_OK;
  if (mlp) {
    // Layer: the attention block first; the MLP body then runs on x1 (fp32)
    if (layer) {
      ee_status s = layer_attn_forward(cfg, B, P, x, n, st);
      if (s != EE_OK) return s;
    }
    const void* xin = layer ? (const void*)B.x1 : (const void*)x;
    // a1: u = RMSNorm_a(x)
    { Prof p_("a1_rmsnorm_fwd", st, 0, 0, (layer ? 6.0 : 4.0) * n * h + 4.0 * n);
    EE_CUDA(launch_rmsnorm_fwd(xin, layer, (const float*)P.g_a, cfg->norm_eps, B.u, B.rx, n, h, st)); }
    // a2: [A|B] = u [W_gate|W_up]^T (paired B tiles), M = silu(A) * B
    {
      GemmArgs a = base_args((int)n, F, h);
      a.ab = B.ab;
      a.ld_ab = 2LL * F;
      a.mact = B.mact;
      a.ld_m = F;
      a.ffn = F;
      Mat A{B.u, n, h, h}, B0{P.w_gate, F, h, h}, B1{P.w_up, F, h, h};
      Prof p_("a2_gateup_swiglu", st, 4.0 * n * F * h, 4.0 * n * F * h, 0);
      EE_CUDA(gemm_run(EPI_SWIGLU_FWD, true, true, A, B0, &B1, B_PAIR, 0, a, st));
    }
    // a3: y = x + M W_down^T  (fp32 residual stream, A15; Layer: y = x1 + ...)
    {
      GemmArgs a = base_args((int)n, h, F);
      a.out0 = B.y;
      a.ldo = h;
      if (layer) {  // fp32 residual: y <- x1, then accumulate
        EE_CUDA(cudaMemcpyAsync(B.y, B.x1, 4 * (size_t)n * h, cudaMemcpyDeviceToDevice, st));
        a.accumulate = 1;
      } else {
        a.resid = x;
        a.ld_resid = h;
      }
      Mat A{B.mact, n, F, F}, Bm{P.w_down, h, F, F};
      Prof p_("a3_down_resid", st, 2.0 * n * F * h, 2.0 * n * F * h, 0);
      EE_CUDA(gemm_run(layer ? EPI_F32 : EPI_RESID, true, true, A, Bm, nullptr, B_PLAIN, 0, a, st));
    }
    // a4: z = RMSNorm_f(y)
    { Prof p_("a4_rmsnorm_fwd", st, 0, 0, 6.0 * n * h + 4.0 * n);
    EE_CUDA(launch_rmsnorm_fwd(B.y, true, (const float*)P.g_f, cfg->norm_eps, z, B.ry, n, h, st,
                               ag)); }
  } else {
    { Prof p_("a4_rmsnorm_fwd", st, 0, 0, 4.0 * n * h + 4.0 * n);
    EE_CUDA(launch_rmsnorm_fwd(x, false, (const float*)P.g_f, cfg->norm_eps, z, B.ry, n, h, st,
                               ag)); }
  }
  return EE_OK;
}

// a5: per-V-tile online-softmax partials of S = z W_out^T (logits never stored).
// a7 strategy (cfg->ds_mode, include/ee.h): EE_DS_RECOMPUTE (default) recomputes
// S with a second GEMM whose epilogue forms dS (the FlashAttention-style
// recompute; logits never in HBM); EE_DS_STORED_P has the a5 epilogue store
// P~ = exp(S - tile max) (fp16) into the dS buffer and a7 is an elementwise pass.
static bool ds_recompute(const ee_head_config* cfg) { return cfg->ds_mode != EE_DS_STORED_P; }

ee_status phase_vocab_stats(const ee_head_config* cfg, const Bufs& B, const ee_head_tensors& P,
                            const __nv_bfloat16* z, long long n, const int32_t* targets,
                            cudaStream_t st, bool store_p = false) {
  const int h = cfg->hidden, Vl = cfg->vocab_end - cfg->vocab_begin;
  GemmArgs a = base_args((int)n, Vl, h);
  a.targets = targets;
  a.vocab_begin = cfg->vocab_begin;
  a.part_m = B.pm;
  a.part_s = B.ps;
  a.part_i = B.pi;
  a.tgt_logit = B.tgt;
  if (store_p && !ds_recompute(cfg)) {
    a.ds = B.ds;
    a.ld_ds = Vl;
  }
  Mat A{z, n, h, h}, Bm{P.w_out, Vl, h, h};
  Prof p_("a5_vocab_ce_stats", st, 2.0 * n * Vl * h, 2.0 * n * Vl * h,
          a.ds ? 2.0 * n * Vl : 0.0);
  EE_CUDA(gemm_run(EPI_CE_STATS, true, true, A, Bm, nullptr, B_PLAIN, 0, a, st));
  return EE_OK;
}

// a7 (dS, recomputed S), a8 (dz = dS W_out, if dz_out) and a9 (dW_out = dS^T z).
ee_status phase_vocab_backward(const ee_head_config* cfg, const Bufs& B, const ee_head_tensors& P,
                               const ee_head_tensors& G, const __nv_bfloat16* z, long long n,
                               const int32_t* targets, int accumulate, float* dz_out,
                               cudaStream_t st, const ee_peer_set* rs = nullptr,
                               const GradScatter* gs = nullptr, const AdamFuse* af = nullptr) {
  const int h = cfg->hidden, Vl = cfg->vocab_end - cfg->vocab_begin;
  if (!ds_recompute(cfg)) {  // a7: dS from the stored P~ (elementwise, in place)
    Prof p_("a7_ds_from_p", st, 0, 0, 4.0 * n * Vl);
    EE_CUDA(launch_ce_ds_from_p(B.ds, Vl, n, B.pm, B.lse, B.coef, targets, cfg->vocab_begin,
                                B.tgt, st));
  } else {
    GemmArgs a = base_args((int)n, Vl, h);
    a.targets = targets;
    a.vocab_begin = cfg->vocab_begin;
    a.lse = B.lse;
    a.coef = B.coef;
    a.ds = B.ds;
    a.ld_ds = Vl;
    Mat A{z, n, h, h}, Bm{P.w_out, Vl, h, h};
    Prof p_("a7_ds_recompute", st, 2.0 * n * Vl * h, 0, 0);
    EE_CUDA(gemm_run(EPI_CE_DS, true, true, A, Bm, nullptr, B_PLAIN, 0, a, st));
  }
  if (dz_out || rs) {  // a8: W_out read MN-major in place
    GemmArgs a = base_args((int)n, h, Vl);
    a.out0 = dz_out;
    a.ldo = h;
    if (rs) {  // fused reduce-scatter: rows to their owners' slot [rank] (include/ee.h)
      a.scat_rows = (int)(n / rs->world);
      for (int q = 0; q < rs->world; ++q)
        a.scat[q] = (float*)rs->ptr[q] + (long long)rs->rank * a.scat_rows * h;
    }
    Mat A{B.ds, n, Vl, Vl}, Bm{P.w_out, Vl, h, h};
    Prof p_("a8_dz", st, 2.0 * n * Vl * h, 2.0 * n * Vl * h, 0);
    EE_CUDA(gemm_run(EPI_F32, true, false, A, Bm, nullptr, B_PLAIN, 0, a, st));
  }
  {  // a9: dW_out^T = z^T dS with z^T K-major (transposed copy), dS MN-major; stored transposed
    { Prof p_("transpose_z", st, 0, 0, 4.0 * n * h);
    EE_CUDA(launch_transpose_bf16(z, B.zT, n, h, B.L.ldT, st)); }
    GemmArgs a = base_args(h, Vl, (int)n);
    a.out0 = (float*)G.w_out;
    a.ldo = h;
    a.n_split = Vl;
    a.accumulate = accumulate;
    if (gs) set_scatter(a, gs, 5, -1);
    if (af) set_adam(a, af, 5, -1);
    Mat A{B.zT, h, n, B.L.ldT}, Bm{B.ds, n, Vl, Vl};
    Prof p_("a9_dw_out", st, 2.0 * n * Vl * h, 2.0 * n * Vl * h, 0);
    EE_CUDA(gemm_run(af ? EPI_F32T_ADAM : EPI_F32T, true, false, A, Bm, nullptr, B_PLAIN, 0, a,
                     st));
  }
  return EE_OK;
}

// a10..a13 on n tokens given dz: dg_f (+ dy, MLP grads, dg_a for MLP exits).
ee_status phase_exit_backward(const ee_head_config* cfg, const Bufs& B, const ee_head_tensors& P,
                              const ee_head_tensors& G, const __nv_bfloat16* x, long long n,
                              const float* dz, int accumulate, cudaStream_t st,
                              int nslots = 1, const GradScatter* gs = nullptr,
                              const AdamFuse* af = nullptr) {
  const int h = cfg->hidden, F = cfg->ffn;
  const bool mlp = cfg->arch >= EE_ARCH_MLP, layer = cfg->arch == EE_ARCH_LAYER;
  if (cfg->arch == EE_ARCH_EMBEDDING) return EE_OK;
  const int nparts = (int)((n + NORM_RPB - 1) / NORM_RPB);
  // a10: final RMSNorm backward -> dg_f (and dy for MLP)
  { Prof p_("a10_rmsnorm_bwd", st, 0, 0, (mlp ? 10.0 : 6.0) * n * h);
  EE_CUDA(launch_rmsnorm_bwd(dz, mlp ? (const void*)B.y : (const void*)x, mlp, B.ry,
                             (const float*)P.g_f, mlp ? B.dy : nullptr, B.dgp, n, h, NORM_RPB,
                             st, nullptr, nslots, (long long)n * h)); }
  { Prof p_("reduce_cols", st, 0, 0, 4.0 * nparts * h);
  EE_CUDA(launch_reduce_cols(B.dgp, nparts, h,
                             gs ? gs->p[4][0] : af ? B.gsc : (float*)G.g_f, accumulate, st)); }
  if (!mlp) return EE_OK;
  // a11: dM = dy W_down; dA = dM B silu'(A), dB = dM silu(A), in place over [A|B]
  {
    GemmArgs a = base_args((int)n, F, h);
    a.ab = B.ab;
    a.ld_ab = 2LL * F;
    a.ffn = F;
    Mat A{B.dy, n, h, h}, Bm{P.w_down, h, F, F};
    Prof p_("a11_dm_swiglu_bwd", st, 2.0 * n * F * h, 2.0 * n * F * h, 0);
    EE_CUDA(gemm_run(EPI_SWIGLU_BWD, true, false, A, Bm, nullptr, B_PLAIN, 0, a, st));
  }
  // a11: dW_down = dy^T M  (after dM, which reads W_down: a fused Adam updates it)
  // dW_down = dy^T M  (A = dy^T K-major copy, B = M MN-major)
  {
    { Prof p_("transpose_dy", st, 0, 0, 4.0 * n * h);
    EE_CUDA(launch_transpose_bf16(B.dy, B.dyT, n, h, B.L.ldT, st)); }
    GemmArgs a = base_args(h, F, (int)n);
    a.out0 = (float*)G.w_down;
    a.ldo = F;
    a.accumulate = accumulate;
    if (gs) set_scatter(a, gs, 3, -1);
    if (af) set_adam(a, af, 3, -1);
    Mat A{B.dyT, h, n, B.L.ldT}, Bm{B.mact, n, F, F};
    Prof p_("a11_dw_down", st, 2.0 * n * F * h, 2.0 * n * F * h, 0);
    EE_CUDA(gemm_run(af ? EPI_F32_ADAM : EPI_F32, true, false, A, Bm, nullptr, B_PLAIN, 0, a,
                     st));
  }
  // a12: du = dA W_gate + dB W_up  (K concatenation over the two weights) -> B.dz.
  // Layer exits only: du feeds dx1 (the attention block's gradient).  An MLP
  // exit needs du only for dg_a = sum_t du_t (.) x^_t, which the dW GEMM below
  // produces from its own accumulators (gain identity, DESIGN.md §3 A28).
  if (layer) {
    GemmArgs a = base_args((int)n, h, 2 * F);
    a.out0 = B.dz;
    a.ldo = h;
    Mat A{B.ab, n, 2LL * F, 2LL * F}, B0{P.w_gate, F, h, h}, B1{P.w_up, F, h, h};
    Prof p_("a12_du", st, 4.0 * n * F * h, 4.0 * n * F * h, 0);
    EE_CUDA(gemm_run(EPI_F32, true, false, A, B0, &B1, B_KSPLIT, F, a, st));
  }
  // a12 (after du, which reads W_gate / W_up): [dW_gate; dW_up]^T = u^T [dA|dB]  (A = u^T K-major copy, B = [dA|dB]
  // MN-major), stored transposed; output columns split at F over the two grads.
  // MLP exits: A = x^T (x^ = x r, RMSNorm without its gain) and the epilogue
  // scales row j by g_a[j] (u = g_a (.) x^) and emits, per 256-column block,
  // sum_f W[f][j] acc[j][f] = the block's share of dg_a[j] (a13 without du).
  const int gblocks = (2 * F + GEMM_BN - 1) / GEMM_BN;
  {
    if (layer) {
      Prof p_("transpose_u", st, 0, 0, 4.0 * n * h);
      EE_CUDA(launch_transpose_bf16(B.u, B.uT, n, h, B.L.ldT, st));
    } else {
      Prof p_("transpose_xhat", st, 0, 0, 4.0 * n * h + 4.0 * n);
      EE_CUDA(launch_transpose_bf16(x, B.uT, n, h, B.L.ldT, st, B.rx));
    }
    GemmArgs a = base_args(h, 2 * F, (int)n);
    if (!layer) {
      a.row_scale = (const float*)P.g_a;
      a.gain_part = B.dgp;
      a.gain_w0 = (const __nv_bfloat16*)P.w_gate;
      a.gain_w1 = (const __nv_bfloat16*)P.w_up;
    }
    a.out0 = (float*)G.w_gate;
    a.out1 = (float*)G.w_up;
    a.n_split = F;
    a.ldo = h;
    a.accumulate = accumulate;
    if (gs) set_scatter(a, gs, 1, 2);
    if (af) set_adam(a, af, 1, 2);
    Mat A{B.uT, h, n, B.L.ldT}, Bm{B.ab, n, 2LL * F, 2LL * F};
    Prof p_("a12_dw_gateup", st, 4.0 * n * F * h, 4.0 * n * F * h, 0);
    EE_CUDA(gemm_run(af ? EPI_F32T_ADAM : EPI_F32T, true, false, A, Bm, nullptr, B_PLAIN, 0, a,
                     st));
  }
  if (layer) {
    // a13 (Layer): dg_a and dx1 = dy + RMSNorm_a^T(du), written over dy in place
    Prof p_("a13_rmsnorm_bwd_resid", st, 0, 0, 14.0 * n * h);
    EE_CUDA(launch_rmsnorm_bwd(B.dz, B.x1, true, B.rx, (const float*)P.g_a, B.dy, B.dgp, n, h,
                               NORM_RPB, st, B.dy));
  }
  // a13: dg_a = column sums of the partials (RMSNorm-backward row blocks for
  // Layer exits, dW-GEMM column blocks for MLP exits; no dx: frozen backbone)
  const int gparts = layer ? nparts : (n > 0 ? gblocks : 0);
  { Prof p_("reduce_cols", st, 0, 0, 4.0 * gparts * h);
  EE_CUDA(launch_reduce_cols(B.dgp, gparts, h,
                             gs ? gs->p[0][0] : af ? B.gsc + h : (float*)G.g_a, accumulate,
                             st)); }
  if (layer) return layer_attn_backward(cfg, B, P, G, x, n, accumulate, st, gs, af, B.gsc + 2 * h);
  return EE_OK;
}

ee_status zero_grads(const ee_head_config* cfg, const ee_head_tensors& G, bool vocab_part,
                     bool exit_part, cudaStream_t st) {
  for (int k = 0; k < NTENS; ++k) {
    void* p = G.*(kTens[k].f);
    const bool is_vocab = kTens[k].vocab;
    if (p && ((is_vocab && vocab_part) || (!is_vocab && exit_part)))
      EE_CUDA(cudaMemsetAsync(p, 0, 4 * (size_t)tensor_numel(cfg, k), st));
  }
  return EE_OK;
}

}  // namespace

extern "C" {

static ee_status tune_step_impl(const ee_head_config* cfg, const void* const* hidden,
                                int64_t n_tokens, const int32_t* targets,
                                const float* exit_weights, const ee_head_tensors* params,
                                ee_head_tensors* grads, const ee_peer_set* arenas,
                                int32_t accumulate, float* loss_out, const ee_step_aux* aux,
                                const int64_t* valid_count, void* workspace, size_t ws_bytes,
                                void* stream, const AdamFuse* afuse = nullptr) {
  ee_status s = check_cfg(cfg);
  if (s != EE_OK) return s;
  if (cfg->vocab_begin != 0 || cfg->vocab_end != cfg->vocab)
    return fail(EE_ERR_ARG, "ee_tune_step needs the full vocabulary; use the ee_vp_* phases "
                            "for a vocab-parallel shard");
  const int E = cfg->num_exits;
  if (!hidden || !exit_weights || !params || (!grads && !arenas && !afuse) || !loss_out ||
      n_tokens < 0 ||
      (n_tokens > 0 && !targets))
    return fail(EE_ERR_ARG, "NULL argument or n_tokens < 0");
  if (n_tokens > (1LL << 30)) return fail(EE_ERR_SHAPE, "n_tokens too large");
  if ((s = check_tokens(cfg, n_tokens)) != EE_OK) return s;
  if (valid_count && cfg->token_weighting == EE_WEIGHT_CONFIDENCE)
    return fail(EE_ERR_UNSUPPORTED, "confidence weighting needs every token of the batch in one "
                                    "call; a DP shard uses EE_WEIGHT_CONFIDENCE_SUM + "
                                    "ee_normalize_exit");
  for (int i = 0; i < E; ++i) {
    if ((s = check_arch_tensors(cfg, params[i], "params", i)) != EE_OK) return s;
    if (!arenas && !afuse && (s = check_arch_tensors(cfg, grads[i], "grads", i)) != EE_OK)
      return s;
    if (arenas) {
      const ee_peer_set& a = arenas[i];
      if (a.world < 1 || a.world > EE_MAX_PEERS || a.rank < 0 || a.rank >= a.world)
        return fail(EE_ERR_ARG, "grad_arenas[%d]: bad rank/world", i);
      for (int q = 0; q < a.world; ++q)
        if (!a.ptr[q] || !aligned16(a.ptr[q]))
          return fail(EE_ERR_ALIGN, "grad_arenas[%d].ptr[%d] NULL or misaligned", i, q);
    }
    if (n_tokens > 0 && (!hidden[i] || !aligned16(hidden[i])))
      return fail(hidden[i] ? EE_ERR_ALIGN : EE_ERR_ARG, "hidden[%d] NULL or misaligned", i);
  }
  if ((targets && !aligned16(targets)) || !aligned16(workspace))
    return fail(EE_ERR_ALIGN, "targets/workspace not 16-byte aligned");
  const long long n = n_tokens;
  const Bufs B = make_bufs(cfg, n, workspace);
  if (!workspace || ws_bytes < B.L.total)
    return fail(EE_ERR_WORKSPACE, "workspace needs %zu bytes, got %zu", B.L.total, ws_bytes);
  if ((s = check_device()) != EE_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;

  { Prof p_("count_valid", st, 0, 0, 4.0 * n);
  EE_CUDA(launch_count_valid(targets, n, cfg->vocab, B.vcount, B.status, st)); }
  const long long* vc = valid_count ? (const long long*)valid_count : B.vcount;

  if (n == 0) {
    for (int i = 0; i < E && !accumulate; ++i) {
      if (!arenas) {
        if ((s = zero_grads(cfg, grads[i], true, true, st)) != EE_OK) return s;
        continue;
      }
      const GradScatter gs = make_scatter(cfg, arenas[i]);   // zero this rank's slots
      for (int k = 0; k < NTENS; ++k) {
        if (!tensor_needed(cfg, k)) continue;
        long long R, C;
        tensor_rc(cfg, k, &R, &C);
        for (int q = 0; q < arenas[i].world; ++q)
          if (shard_rows(R, arenas[i].world, q) > 0)
            EE_CUDA(cudaMemsetAsync(gs.p[k][q], 0, 4 * shard_rows(R, arenas[i].world, q) * C, st));
      }
    }
    EE_CUDA(cudaMemsetAsync(loss_out, 0, sizeof(float) * E, st));
    return EE_OK;
  }
  const bool nrm = cfg->arch != EE_ARCH_EMBEDDING;
  for (int i = 0; i < E; ++i) {
    const ee_head_tensors& P = params[i];
    ee_head_tensors G0;
    memset(&G0, 0, sizeof(G0));
    const ee_head_tensors& G = (arenas || afuse) ? G0 : grads[i];
    GradScatter gsv;
    const GradScatter* gs = nullptr;
    if (arenas) {
      gsv = make_scatter(cfg, arenas[i]);
      gs = &gsv;
    }
    const AdamFuse* af = afuse ? &afuse[i] : nullptr;
    const __nv_bfloat16* x = (const __nv_bfloat16*)hidden[i];
    const __nv_bfloat16* z = nullptr;
    Nvtx nv_exit("ee exit %d", i);
    { Nvtx nv_("exit forward (a1-a4)");
    if ((s = phase_exit_forward(cfg, B, P, x, n, nullptr, &z, st)) != EE_OK) return s; }
    { Nvtx nv_("vocab GEMM + online-softmax stats (a5)");
    if ((s = phase_vocab_stats(cfg, B, P, z, n, targets, st, true)) != EE_OK) return s; }
    // a6: lse, coef, per-token aux, L_i
    {
      const ee_step_aux* ax = aux ? &aux[i] : nullptr;
      const bool dynw = cfg->token_weighting != EE_WEIGHT_UNIFORM;
      const bool norm = cfg->token_weighting != EE_WEIGHT_CONFIDENCE_SUM;
      { Prof p_("a6_ce_finalize", st, 0, 0, 12.0 * B.L.nb * n + 24.0 * n);
      EE_CUDA(launch_ce_finalize(B.pm, B.ps, B.pi, B.tgt, targets, B.L.nb, n, vc,
                                 exit_weights[i], B.lse, B.coef, ax ? ax->lse : nullptr,
                                 ax ? ax->loss_tok : nullptr, ax ? ax->argmax : nullptr,
                                 ax ? ax->conf : nullptr, B.loss_part,
                                 dynw ? B.wsum_part : nullptr, B.L.nfin, st)); }
      { Prof p2_("a6_loss_reduce", st, 0, 0, 4.0 * B.L.nfin);
      EE_CUDA(launch_loss_reduce(B.loss_part, B.L.nfin, vc, dynw ? B.wsum_part : nullptr, B.wsum,
                                 loss_out + i, B.status, i, st, norm)); }
      if (dynw) {
        Prof p3_("a6_coef_scale", st, 0, 0, 8.0 * n);
        EE_CUDA(launch_ce_coef_scale(B.coef, n, exit_weights[i], norm ? B.wsum : nullptr, st));
      }
      if (ax && ax->weight_sum)
        EE_CUDA(cudaMemcpyAsync(ax->weight_sum, B.wsum, sizeof(float), cudaMemcpyDeviceToDevice, st));
    }
    { Nvtx nv_("vocab backward (a7-a9)");
    if ((s = phase_vocab_backward(cfg, B, P, G, z, n, targets, accumulate, nrm ? B.dz : nullptr,
                                  st, nullptr, gs, af)) != EE_OK)
      return s; }
    { Nvtx nv_("exit backward (a10-a13)");
    if ((s = phase_exit_backward(cfg, B, P, G, x, n, B.dz, accumulate, st, 1, gs, af)) != EE_OK)
      return s; }
    if (af) {  // the gains' Adam (their gradients are column sums, in B.gsc)
      const int gk[3] = {4, 0, 6};
      for (int j = 0; j < 3; ++j) {
        const AdamOut& t = af->t[gk[j]];
        if (!tensor_needed(cfg, gk[j])) continue;
        const AdamScal& c = af->sc;
        Prof p_("a15_adam_gain", st, 0, 0, 30.0 * cfg->hidden);
        EE_CUDA(launch_adam(t.th, nullptr, (float*)t.op, B.gsc + (size_t)j * cfg->hidden, t.m,
                            t.v, cfg->hidden, c.lr, c.b1, c.b2, c.eps, c.wd, c.bc1, c.bc2, c.gs,
                            st));
      }
    }
  }
  return EE_OK;
}

ee_status ee_tune_step_adam(const ee_head_config* cfg, const void* const* hidden,
                            int64_t n_tokens, const int32_t* targets, const float* exit_weights,
                            ee_head_tensors* operand, ee_head_tensors* master, ee_head_tensors* m,
                            ee_head_tensors* v, float lr, float beta1, float beta2, float eps,
                            float weight_decay, int64_t step, float grad_scale, float* loss_out,
                            const ee_step_aux* aux, const int64_t* valid_count, void* workspace,
                            size_t ws_bytes, void* stream) {
  ee_status s = check_cfg(cfg);
  if (s != EE_OK) return s;
  if (cfg->token_weighting == EE_WEIGHT_CONFIDENCE_SUM)
    return fail(EE_ERR_UNSUPPORTED, "ee_tune_step_adam: the gradient must be final in the call");
  if (!operand || !master || !m || !v) return fail(EE_ERR_ARG, "NULL parameter state");
  if (step < 1) return fail(EE_ERR_ARG, "step must be >= 1");
  if (n_tokens <= 0) return fail(EE_ERR_SHAPE, "ee_tune_step_adam needs n_tokens > 0");
  const int E = cfg->num_exits;
  if (E > 64) return fail(EE_ERR_SHAPE, "at most 64 exits per call");
  AdamFuse af[64];
  const float bc1 = (float)(1.0 - std::pow((double)beta1, (double)step));
  const float bc2 = (float)(1.0 - std::pow((double)beta2, (double)step));
  for (int i = 0; i < E; ++i) {
    if ((s = check_arch_tensors(cfg, operand[i], "operand", i)) != EE_OK) return s;
    if ((s = check_arch_tensors(cfg, master[i], "master", i)) != EE_OK) return s;
    if ((s = check_arch_tensors(cfg, m[i], "m", i)) != EE_OK) return s;
    if ((s = check_arch_tensors(cfg, v[i], "v", i)) != EE_OK) return s;
    memset(&af[i], 0, sizeof(AdamFuse));
    af[i].sc = AdamScal{lr, beta1, beta2, eps, weight_decay, bc1, bc2, grad_scale};
    for (int k = 0; k < NTENS; ++k) {
      const TInfo& ti = kTens[k];
      if (!tensor_needed(cfg, k)) continue;
      float* th = (float*)(master[i].*(ti.f));
      void* op = operand[i].*(ti.f);
      if (ti.gain && op == (void*)th) op = nullptr;   // gains may alias their master
      af[i].t[k] = AdamOut{th, (float*)(m[i].*(ti.f)), (float*)(v[i].*(ti.f)),
                           (__nv_bfloat16*)op};
    }
  }
  return tune_step_impl(cfg, hidden, n_tokens, targets, exit_weights, operand, nullptr, nullptr,
                        0, loss_out, aux, valid_count, workspace, ws_bytes, stream, af);
}

ee_status ee_tune_step(const ee_head_config* cfg, const void* const* hidden, int64_t n_tokens,
                       const int32_t* targets, const float* exit_weights,
                       const ee_head_tensors* params, ee_head_tensors* grads, int32_t accumulate,
                       float* loss_out, const ee_step_aux* aux, const int64_t* valid_count,
                       void* workspace, size_t ws_bytes, const ee_comm* comm, void* stream) {
  if (comm) {
    ee_status s = check_cfg(cfg);
    if (s != EE_OK) return s;
    if ((s = check_device()) != EE_OK) return s;
    for (int i = 0; i < cfg->num_exits; ++i) {
      if (!params || !grads) return fail(EE_ERR_ARG, "NULL params/grads");
      if ((s = check_arch_tensors(cfg, params[i], "params", i)) != EE_OK) return s;
      if ((s = check_arch_tensors(cfg, grads[i], "grads", i)) != EE_OK) return s;
    }
    return comm_tune_step(comm, cfg, hidden, n_tokens, targets, exit_weights, params, grads,
                          accumulate, loss_out, aux, valid_count, workspace, ws_bytes, stream);
  }
  return tune_step_impl(cfg, hidden, n_tokens, targets, exit_weights, params, grads, nullptr,
                        accumulate, loss_out, aux, valid_count, workspace, ws_bytes, stream);
}

ee_status ee_tune_step_rs(const ee_head_config* cfg, const void* const* hidden, int64_t n_tokens,
                          const int32_t* targets, const float* exit_weights,
                          const ee_head_tensors* params, const ee_peer_set* grad_arenas,
                          float* loss_out, const ee_step_aux* aux, const int64_t* valid_count,
                          void* workspace, size_t ws_bytes, void* stream) {
  if (!grad_arenas) return fail(EE_ERR_ARG, "grad_arenas required");
  if (cfg && cfg->token_weighting == EE_WEIGHT_CONFIDENCE)
    return fail(EE_ERR_UNSUPPORTED, "ee_tune_step_rs: the confidence normaliser spans the ranks; "
                                    "use EE_WEIGHT_CONFIDENCE_SUM + grad_divisor");
  return tune_step_impl(cfg, hidden, n_tokens, targets, exit_weights, params, nullptr,
                        grad_arenas, 0, loss_out, aux, valid_count, workspace, ws_bytes, stream);
}

ee_status ee_dp_shard_layout(const ee_head_config* cfg, int32_t world, int32_t rank,
                             int32_t tensor, int64_t* row_begin, int64_t* rows,
                             int64_t* arena_offset_floats, int64_t* arena_total_floats) {
  ee_status s = check_cfg(cfg);
  if (s != EE_OK) return s;
  if (world < 1 || world > EE_MAX_PEERS || rank < 0 || rank >= world || tensor < 0 ||
      tensor >= NTENS || !row_begin || !rows || !arena_offset_floats || !arena_total_floats)
    return fail(EE_ERR_ARG, "bad ee_dp_shard_layout arguments");
  long long R, C;
  tensor_rc(cfg, tensor, &R, &C);
  const bool need = tensor_needed(cfg, tensor);
  *row_begin = need ? std::min<long long>(R, (long long)rank * shard_chunk(R, world)) : 0;
  *rows = need ? shard_rows(R, world, rank) : 0;
  *arena_offset_floats = arena_offset(cfg, world, rank, tensor);
  *arena_total_floats = arena_offset(cfg, world, rank, NTENS);
  return EE_OK;
}

// ---------------------------------------------------------------- backbone partial forward
static ee_status check_backbone(const ee_backbone_config* c) {
  if (!c) return fail(EE_ERR_ARG, "backbone cfg is NULL");
  if (c->n_heads < 1 || c->n_kv_heads < 1 || c->n_heads % c->n_kv_heads != 0)
    return fail(EE_ERR_SHAPE, "n_kv_heads must divide n_heads");
  if (c->hidden != c->n_heads * 128 || c->hidden > 16384)
    return fail(EE_ERR_SHAPE, "hidden must be n_heads * 128 (head dim 128)");
  if (c->ffn < 128 || c->ffn % 128 != 0) return fail(EE_ERR_SHAPE, "ffn must be a multiple of 128");
  if (c->seq_len < 64 || c->seq_len % 64 != 0)
    return fail(EE_ERR_SHAPE, "seq_len must be a positive multiple of 64");
  if (!(c->norm_eps >= 0.f) || !(c->rope_theta > 0.f)) return fail(EE_ERR_ARG, "bad eps/theta");
  return EE_OK;
}

struct BbLayout {
  size_t x, u, q, k, v, o, ab, m, r, rope, total;
};
static BbLayout bb_layout(const ee_backbone_config* c, long long n) {
  BbLayout L{};
  const long long h = c->hidden, hkv = 128LL * c->n_kv_heads, F = c->ffn;
  size_t off = 0;
  auto take = [&](size_t b) {
    size_t r = off;
    off = align_up(off + b);
    return r;
  };
  L.x = take(4 * (size_t)n * h);
  L.u = take(2 * (size_t)n * h);
  L.q = take(2 * (size_t)n * h);
  L.k = take(2 * (size_t)n * hkv);
  L.v = take(2 * (size_t)n * hkv);
  L.o = take(2 * (size_t)n * h);
  L.ab = take(2 * (size_t)n * 2 * F);
  L.m = take(2 * (size_t)n * F);
  L.r = take(4 * (size_t)(n > 0 ? n : 1));
  L.rope = take(8 * 64 * (size_t)c->seq_len);
  L.total = off;
  return L;
}

ee_status ee_backbone_workspace_size(const ee_backbone_config* cfg, int64_t n_tokens,
                                     size_t* bytes) {
  ee_status s = check_backbone(cfg);
  if (s != EE_OK) return s;
  if (!bytes || n_tokens < 0) return fail(EE_ERR_ARG, "bytes NULL or n_tokens < 0");
  *bytes = bb_layout(cfg, n_tokens).total;
  return EE_OK;
}

ee_status ee_backbone_forward(const ee_backbone_config* cfg, const ee_layer_tensors* layers,
                              int32_t n_layers, const void* x0, int64_t n_tokens,
                              const int32_t* exit_after, int32_t num_exits,
                              void* const* hidden_out, void* workspace, size_t ws_bytes,
                              void* stream) {
  ee_status s = check_backbone(cfg);
  if (s != EE_OK) return s;
  if (!layers || !x0 || !exit_after || !hidden_out || num_exits < 1 || n_tokens < 0)
    return fail(EE_ERR_ARG, "NULL argument");
  if (n_tokens % cfg->seq_len != 0)
    return fail(EE_ERR_SHAPE, "n_tokens must be a multiple of seq_len");
  for (int i = 0; i < num_exits; ++i) {
    if (exit_after[i] < 1 || exit_after[i] > n_layers || (i && exit_after[i] <= exit_after[i - 1]))
      return fail(EE_ERR_ARG, "exit_after must be ascending in [1, n_layers]");
    if (!hidden_out[i]) return fail(EE_ERR_ARG, "hidden_out[%d] is NULL", i);
  }
  const int last = exit_after[num_exits - 1];
  for (int l = 0; l < last; ++l) {
    const ee_layer_tensors& t = layers[l];
    const void* ps[9] = {t.g_att, t.w_q, t.w_k, t.w_v, t.w_o, t.g_mlp, t.w_gate, t.w_up, t.w_down};
    for (const void* p : ps)
      if (!p || !aligned16(p)) return fail(EE_ERR_ARG, "layer %d: tensor NULL or misaligned", l + 1);
  }
  const long long n = n_tokens;
  const BbLayout L = bb_layout(cfg, n);
  if (!workspace || !aligned16(workspace) || ws_bytes < L.total)
    return fail(EE_ERR_WORKSPACE, "workspace needs %zu bytes, got %zu", L.total, ws_bytes);
  if ((s = check_device()) != EE_OK) return s;
  if (n == 0) return EE_OK;
  cudaStream_t st = (cudaStream_t)stream;
  uint8_t* ws = (uint8_t*)workspace;
  float* x = (float*)(ws + L.x);
  __nv_bfloat16* u = (__nv_bfloat16*)(ws + L.u);
  __nv_bfloat16* q = (__nv_bfloat16*)(ws + L.q);
  __nv_bfloat16* k = (__nv_bfloat16*)(ws + L.k);
  __nv_bfloat16* v = (__nv_bfloat16*)(ws + L.v);
  __nv_bfloat16* o = (__nv_bfloat16*)(ws + L.o);
  __nv_bfloat16* ab = (__nv_bfloat16*)(ws + L.ab);
  __nv_bfloat16* mact = (__nv_bfloat16*)(ws + L.m);
  float* r = (float*)(ws + L.r);
  float2* rope = (float2*)(ws + L.rope);
  EE_CUDA(launch_rope_table(rope, cfg->seq_len, cfg->rope_theta, st));
  const int h = cfg->hidden, Hq = cfg->n_heads, Hkv = cfg->n_kv_heads, F = cfg->ffn;
  const int hkv = 128 * Hkv;
  { Prof p_("bb_cast_in", st, 0, 0, 6.0 * n * h);
  EE_CUDA(launch_cast_bf16_f32((const __nv_bfloat16*)x0, x, n * h, st)); }
  int next_exit = 0;
  for (int l = 0; l < last; ++l) {
    const ee_layer_tensors& t = layers[l];
    { Prof p_("bb_rmsnorm_att", st, 0, 0, 6.0 * n * h);
    EE_CUDA(launch_rmsnorm_fwd(x, true, (const float*)t.g_att, cfg->norm_eps, u, r, n, h, st)); }
    struct Proj {
      const void* w;
      __nv_bfloat16* out;
      int N;
      const char* name;
    } projs[3] = {{t.w_q, q, h, "bb_q_proj"}, {t.w_k, k, hkv, "bb_k_proj"}, {t.w_v, v, hkv, "bb_v_proj"}};
    for (int j = 0; j < 3; ++j) {  // RoPE fused into the q / k epilogues
      const Proj& pj = projs[j];
      GemmArgs a = base_args((int)n, pj.N, h);
      a.outb = pj.out;
      a.ldo = pj.N;
      if (j < 2) {
        a.rope_seq = cfg->seq_len;
        a.rope_theta = cfg->rope_theta;
        a.rope_tab = rope;
      }
      Mat A{u, n, h, h}, B{pj.w, pj.N, h, h};
      Prof p_(pj.name, st, 2.0 * n * pj.N * h, 2.0 * n * pj.N * h, 0);
      EE_CUDA(gemm_run(EPI_BF16, true, true, A, B, nullptr, B_PLAIN, 0, a, st));
    }
    { const double fl = 2.0 * 2.0 * (double)n * (cfg->seq_len + 64) / 2.0 * h;  // causal
      Prof p_("bb_attention", st, fl, fl, 0);
      EE_CUDA(attn_forward(q, k, v, o, n, cfg->seq_len, Hq, Hkv, nullptr, st)); }
    {  // x += o W_o^T
      GemmArgs a = base_args((int)n, h, h);
      a.out0 = x;
      a.ldo = h;
      a.accumulate = 1;
      Mat A{o, n, h, h}, B{t.w_o, h, h, h};
      Prof p_("bb_o_proj", st, 2.0 * n * h * h, 2.0 * n * h * h, 0);
      EE_CUDA(gemm_run(EPI_F32, true, true, A, B, nullptr, B_PLAIN, 0, a, st));
    }
    { Prof p_("bb_rmsnorm_mlp", st, 0, 0, 6.0 * n * h);
    EE_CUDA(launch_rmsnorm_fwd(x, true, (const float*)t.g_mlp, cfg->norm_eps, u, r, n, h, st)); }
    {
      GemmArgs a = base_args((int)n, F, h);
      a.ab = ab;
      a.ld_ab = 2LL * F;
      a.mact = mact;
      a.ld_m = F;
      a.ffn = F;
      Mat A{u, n, h, h}, B0{t.w_gate, F, h, h}, B1{t.w_up, F, h, h};
      Prof p_("bb_gateup_swiglu", st, 4.0 * n * F * h, 4.0 * n * F * h, 0);
      EE_CUDA(gemm_run(EPI_SWIGLU_FWD, true, true, A, B0, &B1, B_PAIR, 0, a, st));
    }
    {  // x += M W_down^T
      GemmArgs a = base_args((int)n, h, F);
      a.out0 = x;
      a.ldo = h;
      a.accumulate = 1;
      Mat A{mact, n, F, F}, B{t.w_down, h, F, F};
      Prof p_("bb_down", st, 2.0 * n * F * h, 2.0 * n * F * h, 0);
      EE_CUDA(gemm_run(EPI_F32, true, true, A, B, nullptr, B_PLAIN, 0, a, st));
    }
    if (l + 1 == exit_after[next_exit]) {
      Prof p_("bb_cast_out", st, 0, 0, 6.0 * n * h);
      EE_CUDA(launch_cast_f32_bf16(x, (__nv_bfloat16*)hidden_out[next_exit], n * h, st));
      ++next_exit;
    }
  }
  return EE_OK;
}

// ---------------------------------------------------------------- early-exit inference
// Decode shapes (n <= SKINNY_MAX_M tokens): the exit head streams its weights
// through the skinny kernels (skinny.cu); the CE partials of the 32-column
// vocab blocks go to the dS region of the workspace (unused at inference).
static ee_status infer_decode_exit(const ee_head_config* cfg, const Bufs& B,
                                   const ee_head_tensors& P, const __nv_bfloat16* x, long long n,
                                   float* pm, float* ps, int32_t* pi, cudaStream_t st) {
  const int h = cfg->hidden, F = cfg->ffn, Vl = cfg->vocab_end - cfg->vocab_begin;
  const int M = (int)n;
  const __nv_bfloat16* z = x;
  if (cfg->arch != EE_ARCH_EMBEDDING) {
    const void* yin = x;
    bool yf32 = false;
    if (cfg->arch == EE_ARCH_MLP) {
      { Prof p_("dec_rmsnorm_a", st, 0, 0, 4.0 * n * h + 4.0 * h);
      EE_CUDA(launch_rmsnorm_fwd(x, false, (const float*)P.g_a, cfg->norm_eps, B.u, B.rx, n, h, st,
                                 nullptr, true)); }
      {
        SkinnyArgs a{};
        a.x = B.u; a.ldx = h; a.st = B.status; a.W0 = (const __nv_bfloat16*)P.w_gate;
        a.W1 = (const __nv_bfloat16*)P.w_up; a.K = h; a.N = F; a.outb = B.mact; a.ldo = F;
        Prof p_("dec_gateup_swiglu", st, 4.0 * n * F * h, 4.0 * n * F * h, 4.0 * F * h);
        EE_CUDA(launch_skinny(SK_SWIGLU, a, M, st));
      }
      {
        SkinnyArgs a{};
        a.x = B.mact; a.ldx = F; a.st = B.status; a.W0 = (const __nv_bfloat16*)P.w_down; a.K = F; a.N = h;
        a.out = B.y; a.ldo = h; a.resid = x; a.ldr = h;
        Prof p_("dec_down_resid", st, 2.0 * n * F * h, 2.0 * n * F * h, 2.0 * F * h);
        EE_CUDA(launch_skinny(SK_RESID, a, M, st));
      }
      yin = B.y;
      yf32 = true;
    }
    { Prof p_("dec_rmsnorm_f", st, 0, 0, 4.0 * n * h + 4.0 * h);
    EE_CUDA(launch_rmsnorm_fwd(yin, yf32, (const float*)P.g_f, cfg->norm_eps, B.z, B.ry, n, h, st,
                               nullptr, true)); }
    z = B.z;
  }
  SkinnyArgs a{};
  a.x = z; a.ldx = h; a.st = B.status; a.W0 = (const __nv_bfloat16*)P.w_out; a.K = h; a.N = Vl;
  a.pm = pm; a.ps = ps; a.pi = pi; a.vocab_begin = cfg->vocab_begin;
  Prof p_("dec_vocab_ce", st, 2.0 * n * Vl * h, 2.0 * n * Vl * h, 2.0 * Vl * h);
  EE_CUDA(launch_skinny(SK_CE, a, M, st));
  return EE_OK;
}

// Confidence-based exit decision: per exit, the greedy token and
// the max softmax probability; first_exit[t] = lowest exit with c >= tau.
ee_status ee_exit_infer(const ee_head_config* cfg, const void* const* hidden, int64_t n_tokens,
                        const ee_head_tensors* params, float threshold, int32_t* const* argmax_out,
                        float* const* conf_out, int32_t* first_exit, void* workspace,
                        size_t ws_bytes, void* stream) {
  ee_status s = check_cfg(cfg);
  if (s != EE_OK) return s;
  if (cfg->vocab_begin != 0 || cfg->vocab_end != cfg->vocab)
    return fail(EE_ERR_ARG, "ee_exit_infer needs the full vocabulary");
  const int E = cfg->num_exits;
  if (!hidden || !params || !argmax_out || !conf_out || n_tokens < 0)
    return fail(EE_ERR_ARG, "NULL argument or n_tokens < 0");
  if (E > 64) return fail(EE_ERR_SHAPE, "at most 64 exits");
  if ((s = check_tokens(cfg, n_tokens)) != EE_OK) return s;
  for (int i = 0; i < E; ++i) {
    if ((s = check_arch_tensors(cfg, params[i], "params", i)) != EE_OK) return s;
    if (n_tokens > 0 && (!hidden[i] || !argmax_out[i] || !conf_out[i]))
      return fail(EE_ERR_ARG, "exit %d: NULL hidden/output", i);
  }
  const long long n = n_tokens;
  const Bufs B = make_bufs(cfg, n, workspace);
  if (!workspace || !aligned16(workspace) || ws_bytes < B.L.total)
    return fail(EE_ERR_WORKSPACE, "workspace needs %zu bytes, got %zu", B.L.total, ws_bytes);
  if ((s = check_device()) != EE_OK) return s;
  if (n == 0) return EE_OK;
  cudaStream_t st = (cudaStream_t)stream;
  // no targets at inference: every row "ignored" (the int32 -1 pattern)
  int32_t* no_targets = (int32_t*)B.tgt;  // tgt (fp32 [n]) is free: no target logits needed
  EE_CUDA(cudaMemsetAsync(no_targets, 0xFF, sizeof(int32_t) * n, st));
  EE_CUDA(cudaMemsetAsync(B.vcount, 0, sizeof(long long), st));
  static const int skinny_env = [] {
    const char* e = getenv("EE_INFER_SKINNY");
    return e ? atoi(e) : 1;
  }();
  const bool decode = skinny_env && n <= SKINNY_MAX_M && cfg->arch != EE_ARCH_LAYER;
  for (int i = 0; i < E; ++i) {
    const __nv_bfloat16* x = (const __nv_bfloat16*)hidden[i];
    if (decode) {
      const int nbd = skinny_blocks(cfg->vocab_end - cfg->vocab_begin);
      float* pm = (float*)B.ds;
      float* ps = pm + (size_t)nbd * n;
      int32_t* pi = (int32_t*)(ps + (size_t)nbd * n);
      if ((s = infer_decode_exit(cfg, B, params[i], x, n, pm, ps, pi, st)) != EE_OK) return s;
      Prof p_("infer_finalize", st, 0, 0, 12.0 * nbd * n + 8.0 * n);
      EE_CUDA(launch_infer_finalize_wide(pm, ps, pi, nbd, (int)n, B.lse, argmax_out[i],
                                         conf_out[i], st));
      continue;
    }
    const __nv_bfloat16* z = nullptr;
    if ((s = phase_exit_forward(cfg, B, params[i], x, n, nullptr, &z, st)) != EE_OK) return s;
    if ((s = phase_vocab_stats(cfg, B, params[i], z, n, no_targets, st)) != EE_OK) return s;
    Prof p_("infer_finalize", st, 0, 0, 12.0 * B.L.nb * n + 8.0 * n);
    EE_CUDA(launch_ce_finalize(B.pm, B.ps, B.pi, nullptr, no_targets, B.L.nb, n, B.vcount, 0.f,
                               B.lse, B.coef, nullptr, nullptr, argmax_out[i], conf_out[i],
                               B.loss_part, nullptr, B.L.nfin, st));
  }
  if (first_exit) {
    float* confs[64];
    for (int i = 0; i < E; ++i) confs[i] = conf_out[i];
    Prof p_("infer_first_exit", st, 0, 0, 4.0 * E * n + 4.0 * n);
    EE_CUDA(launch_first_exit((const float* const*)confs, E, n, threshold, first_exit, st));
  }
  return EE_OK;
}

// ---------------------------------------------------------------- vocab parallel
// One exit, one rank of P.  The caller runs the collectives between phases
// (include/ee.h, "vocab-parallel phases").  cfg->num_exits is ignored (the
// calls take one exit's tensors); the workspace is sized for n_all tokens.
static ee_status vp_common(const ee_head_config* cfg, long long n_all, void* ws, size_t ws_bytes,
                           Bufs* B) {
  ee_status s = check_cfg(cfg);
  if (s != EE_OK) return s;
  if (n_all < 0 || n_all > (1LL << 30)) return fail(EE_ERR_SHAPE, "bad n_all");
  if (!ws || !aligned16(ws)) return fail(EE_ERR_ARG, "workspace NULL or misaligned");
  *B = make_bufs(cfg, n_all, ws);
  if (ws_bytes < B->L.total)
    return fail(EE_ERR_WORKSPACE, "workspace needs %zu bytes, got %zu", B->L.total, ws_bytes);
  return check_device();
}

ee_status ee_vp_exit_forward(const ee_head_config* cfg, const void* hidden, int64_t n_local,
                             int64_t n_all, const ee_head_tensors* params, void* z_out,
                             void* workspace, size_t ws_bytes, void* stream) {
  Bufs B;
  ee_status s = vp_common(cfg, n_all, workspace, ws_bytes, &B);
  if (s != EE_OK) return s;
  if (!params || !z_out || n_local < 0 || n_local > n_all || (n_local > 0 && !hidden))
    return fail(EE_ERR_ARG, "bad ee_vp_exit_forward arguments");
  if (ee_status s2 = check_tokens(cfg, n_local); s2 != EE_OK) return s2;
  if ((s = check_arch_tensors(cfg, *params, "params", 0)) != EE_OK) return s;
  if (!aligned16(z_out) || (hidden && !aligned16(hidden))) return fail(EE_ERR_ALIGN, "misaligned");
  const __nv_bfloat16* z = nullptr;
  return phase_exit_forward(cfg, B, *params, (const __nv_bfloat16*)hidden, n_local,
                            (__nv_bfloat16*)z_out, &z, (cudaStream_t)stream);
}

ee_status ee_vp_vocab_stats(const ee_head_config* cfg, const void* z_all, int64_t n_all,
                            const int32_t* targets_all, const ee_head_tensors* params,
                            int64_t* key_out, float* sums_out, void* workspace, size_t ws_bytes,
                            void* stream) {
  Bufs B;
  ee_status s = vp_common(cfg, n_all, workspace, ws_bytes, &B);
  if (s != EE_OK) return s;
  if (!params || !params->w_out || (n_all > 0 && (!z_all || !targets_all || !key_out || !sums_out)))
    return fail(EE_ERR_ARG, "bad ee_vp_vocab_stats arguments");
  cudaStream_t st = (cudaStream_t)stream;
  if (n_all == 0) return EE_OK;
  { Prof p_("count_valid", st, 0, 0, 4.0 * n_all);
  EE_CUDA(launch_count_valid(targets_all, n_all, cfg->vocab, B.vcount, B.status, st)); }
  if ((s = phase_vocab_stats(cfg, B, *params, (const __nv_bfloat16*)z_all, n_all, targets_all,
                             st, true)) != EE_OK)
    return s;
  Prof p_("vp_local_merge", st, 0, 0, 12.0 * B.L.nb * n_all + 20.0 * n_all);
  EE_CUDA(launch_vp_local_merge(B.pm, B.ps, B.pi, B.tgt, targets_all, B.L.nb, n_all,
                                cfg->vocab_begin, cfg->vocab_end, (long long*)key_out, B.m_loc,
                                sums_out, st));
  return EE_OK;
}

ee_status ee_vp_rescale(const ee_head_config* cfg, int64_t n_all, const int64_t* key_global,
                        float* sums, void* workspace, size_t ws_bytes, void* stream) {
  Bufs B;
  ee_status s = vp_common(cfg, n_all, workspace, ws_bytes, &B);
  if (s != EE_OK) return s;
  if (n_all > 0 && (!key_global || !sums)) return fail(EE_ERR_ARG, "NULL argument");
  if (n_all == 0) return EE_OK;
  cudaStream_t st = (cudaStream_t)stream;
  Prof p_("vp_rescale", st, 0, 0, 20.0 * n_all);
  EE_CUDA(launch_vp_rescale((const long long*)key_global, B.m_loc, sums, n_all, st));
  return EE_OK;
}

static ee_status check_peer_set(const ee_peer_set* p, long long n_all, const char* what) {
  if (!p || p->world < 1 || p->world > EE_MAX_PEERS || p->rank < 0 || p->rank >= p->world)
    return fail(EE_ERR_ARG, "%s: bad ee_peer_set (rank/world)", what);
  for (int q = 0; q < p->world; ++q)
    if (!p->ptr[q] || !aligned16(p->ptr[q]))
      return fail(EE_ERR_ALIGN, "%s: peer pointer %d NULL or misaligned", what, q);
  if (n_all % p->world) return fail(EE_ERR_SHAPE, "%s: n_all not a multiple of world", what);
  return EE_OK;
}

static ee_status vp_vocab_backward_impl(const ee_head_config* cfg, const void* z_all,
                                        int64_t n_all, const int32_t* targets_all,
                                        const int64_t* key_global, const float* sums_global,
                                        float exit_weight, const int64_t* valid_count,
                                        const ee_head_tensors* params, ee_head_tensors* grads,
                                        int32_t accumulate, float* dz_partial,
                                        const ee_peer_set* rs, float* loss_out,
                                        const ee_step_aux* aux, int32_t exit_index,
                                        void* workspace, size_t ws_bytes, void* stream) {
  Bufs B;
  ee_status s = vp_common(cfg, n_all, workspace, ws_bytes, &B);
  if (s != EE_OK) return s;
  if (!params || !grads || !grads->w_out || !loss_out ||
      (n_all > 0 && (!z_all || !targets_all || !key_global || !sums_global)))
    return fail(EE_ERR_ARG, "bad ee_vp_vocab_backward arguments");
  const bool nrm = cfg->arch != EE_ARCH_EMBEDDING;
  if (nrm && n_all > 0 && !dz_partial && !rs) return fail(EE_ERR_ARG, "dz_partial required");
  if (rs && (s = check_peer_set(rs, n_all, "dz_slots")) != EE_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  if (n_all == 0) {
    if (!accumulate && (s = zero_grads(cfg, *grads, true, false, st)) != EE_OK) return s;
    EE_CUDA(cudaMemsetAsync(loss_out, 0, sizeof(float), st));
    return EE_OK;
  }
  const long long* vc = valid_count ? (const long long*)valid_count : B.vcount;
  const bool dynw = cfg->token_weighting != EE_WEIGHT_UNIFORM;
  const bool norm = cfg->token_weighting != EE_WEIGHT_CONFIDENCE_SUM;
  {
    Prof p_("vp_finalize", st, 0, 0, 28.0 * n_all);
    EE_CUDA(launch_vp_finalize((const long long*)key_global, sums_global, targets_all, n_all, vc,
                               exit_weight, B.lse, B.coef, aux ? aux->lse : nullptr,
                               aux ? aux->loss_tok : nullptr, aux ? aux->argmax : nullptr,
                               aux ? aux->conf : nullptr, B.loss_part,
                               dynw ? B.wsum_part : nullptr, B.L.nfin, st));
  }
  {
    Prof p_("a6_loss_reduce", st, 0, 0, 4.0 * B.L.nfin);
    EE_CUDA(launch_loss_reduce(B.loss_part, B.L.nfin, vc, dynw ? B.wsum_part : nullptr, B.wsum,
                               loss_out, B.status, exit_index, st, norm));
  }
  if (dynw) {
    Prof p_("a6_coef_scale", st, 0, 0, 8.0 * n_all);
    EE_CUDA(launch_ce_coef_scale(B.coef, n_all, exit_weight, norm ? B.wsum : nullptr, st));
  }
  if (aux && aux->weight_sum)
    EE_CUDA(cudaMemcpyAsync(aux->weight_sum, B.wsum, sizeof(float), cudaMemcpyDeviceToDevice, st));
  return phase_vocab_backward(cfg, B, *params, *grads, (const __nv_bfloat16*)z_all, n_all,
                              targets_all, accumulate, nrm ? dz_partial : nullptr, st,
                              nrm ? rs : nullptr);
}

ee_status ee_vp_vocab_backward(const ee_head_config* cfg, const void* z_all, int64_t n_all,
                               const int32_t* targets_all, const int64_t* key_global,
                               const float* sums_global, float exit_weight,
                               const int64_t* valid_count, const ee_head_tensors* params,
                               ee_head_tensors* grads, int32_t accumulate, float* dz_partial,
                               float* loss_out, const ee_step_aux* aux, int32_t exit_index,
                               void* workspace, size_t ws_bytes, void* stream) {
  return vp_vocab_backward_impl(cfg, z_all, n_all, targets_all, key_global, sums_global,
                                exit_weight, valid_count, params, grads, accumulate, dz_partial,
                                nullptr, loss_out, aux, exit_index, workspace, ws_bytes, stream);
}

ee_status ee_vp_vocab_backward_rs(const ee_head_config* cfg, const void* z_all, int64_t n_all,
                                  const int32_t* targets_all, const int64_t* key_global,
                                  const float* sums_global, float exit_weight,
                                  const int64_t* valid_count, const ee_head_tensors* params,
                                  ee_head_tensors* grads, int32_t accumulate,
                                  const ee_peer_set* dz_slots, float* loss_out,
                                  const ee_step_aux* aux, int32_t exit_index, void* workspace,
                                  size_t ws_bytes, void* stream) {
  if (!dz_slots) return fail(EE_ERR_ARG, "dz_slots required");
  return vp_vocab_backward_impl(cfg, z_all, n_all, targets_all, key_global, sums_global,
                                exit_weight, valid_count, params, grads, accumulate, nullptr,
                                dz_slots, loss_out, aux, exit_index, workspace, ws_bytes, stream);
}

ee_status ee_vp_exit_backward(const ee_head_config* cfg, const void* hidden, int64_t n_local,
                              int64_t n_all, const ee_head_tensors* params, const float* dz_local,
                              ee_head_tensors* grads, int32_t accumulate, void* workspace,
                              size_t ws_bytes, void* stream) {
  Bufs B;
  ee_status s = vp_common(cfg, n_all, workspace, ws_bytes, &B);
  if (s != EE_OK) return s;
  if (!params || !grads || n_local < 0 || n_local > n_all ||
      (n_local > 0 && cfg->arch != EE_ARCH_EMBEDDING && (!hidden || !dz_local)))
    return fail(EE_ERR_ARG, "bad ee_vp_exit_backward arguments");
  if (ee_status s2 = check_tokens(cfg, n_local); s2 != EE_OK) return s2;
  cudaStream_t st = (cudaStream_t)stream;
  if (n_local == 0) {
    if (!accumulate) return zero_grads(cfg, *grads, false, true, st);
    return EE_OK;
  }
  return phase_exit_backward(cfg, B, *params, *grads, (const __nv_bfloat16*)hidden, n_local,
                             dz_local, accumulate, st);
}

ee_status ee_vp_exit_forward_ag(const ee_head_config* cfg, const void* hidden, int64_t n_local,
                                int64_t n_all, const ee_head_tensors* params,
                                const ee_peer_set* z_all, void* workspace, size_t ws_bytes,
                                void* stream) {
  Bufs B;
  ee_status s = vp_common(cfg, n_all, workspace, ws_bytes, &B);
  if (s != EE_OK) return s;
  if (!params || n_local < 0 || (n_local > 0 && !hidden))
    return fail(EE_ERR_ARG, "bad ee_vp_exit_forward_ag arguments");
  if ((s = check_peer_set(z_all, n_all, "z_all")) != EE_OK) return s;
  if (n_local * z_all->world != n_all) return fail(EE_ERR_SHAPE, "n_all != world * n_local");
  if (ee_status s2 = check_tokens(cfg, n_local); s2 != EE_OK) return s2;
  if ((s = check_arch_tensors(cfg, *params, "params", 0)) != EE_OK) return s;
  if (hidden && !aligned16(hidden)) return fail(EE_ERR_ALIGN, "misaligned");
  PeerRows ag{};
  ag.n = z_all->world;
  ag.row_off = (long long)z_all->rank * n_local;
  for (int q = 0; q < z_all->world; ++q) ag.p[q] = (__nv_bfloat16*)z_all->ptr[q];
  const __nv_bfloat16* z = nullptr;
  return phase_exit_forward(cfg, B, *params, (const __nv_bfloat16*)hidden, n_local, nullptr, &z,
                            (cudaStream_t)stream, &ag);
}

ee_status ee_vp_exit_backward_slots(const ee_head_config* cfg, const void* hidden,
                                    int64_t n_local, int64_t n_all,
                                    const ee_head_tensors* params, const float* dz_slots,
                                    int32_t n_slots, ee_head_tensors* grads, int32_t accumulate,
                                    const ee_peer_set* grad_arenas, void* workspace,
                                    size_t ws_bytes, void* stream) {
  if (n_slots < 1 || n_slots > EE_MAX_PEERS) return fail(EE_ERR_ARG, "n_slots out of range");
  if (dz_slots && !aligned16(dz_slots)) return fail(EE_ERR_ALIGN, "dz_slots misaligned");
  Bufs B;
  ee_status s = vp_common(cfg, n_all, workspace, ws_bytes, &B);
  if (s != EE_OK) return s;
  if (!params || (!grads && !grad_arenas) || n_local < 0 || n_local > n_all ||
      (n_local > 0 && cfg->arch != EE_ARCH_EMBEDDING && (!hidden || !dz_slots)))
    return fail(EE_ERR_ARG, "bad ee_vp_exit_backward_slots arguments");
  if (grad_arenas) {
    const ee_peer_set& a = *grad_arenas;
    if (a.world < 1 || a.world > EE_MAX_PEERS || a.rank < 0 || a.rank >= a.world)
      return fail(EE_ERR_ARG, "grad_arenas: bad rank/world");
    for (int q = 0; q < a.world; ++q)
      if (!a.ptr[q] || !aligned16(a.ptr[q]))
        return fail(EE_ERR_ALIGN, "grad_arenas.ptr[%d] NULL or misaligned", q);
    if (accumulate) return fail(EE_ERR_ARG, "grad_arenas: accumulate must be 0");
  }
  if (ee_status s2 = check_tokens(cfg, n_local); s2 != EE_OK) return s2;
  cudaStream_t st = (cudaStream_t)stream;
  if (n_local == 0) {
    if (grad_arenas) return fail(EE_ERR_SHAPE, "grad_arenas need n_local > 0");
    if (!accumulate) return zero_grads(cfg, *grads, false, true, st);
    return EE_OK;
  }
  ee_head_tensors G0;
  memset(&G0, 0, sizeof(G0));
  GradScatter gsv;
  if (grad_arenas) gsv = make_scatter(cfg, *grad_arenas);
  return phase_exit_backward(cfg, B, *params, grad_arenas ? G0 : *grads,
                             (const __nv_bfloat16*)hidden, n_local, dz_slots, accumulate, st,
                             n_slots, grad_arenas ? &gsv : nullptr);
}

ee_status ee_peer_barrier(const ee_peer_set* signals, uint32_t epoch, void* workspace,
                          void* stream) {
  if (!workspace || !aligned16(workspace)) return fail(EE_ERR_ARG, "workspace NULL or misaligned");
  if (!signals || signals->world < 1 || signals->world > EE_MAX_PEERS || signals->rank < 0 ||
      signals->rank >= signals->world)
    return fail(EE_ERR_ARG, "bad ee_peer_set");
  for (int q = 0; q < signals->world; ++q)
    if (!signals->ptr[q]) return fail(EE_ERR_ARG, "signal pointer %d NULL", q);
  if (ee_status s = check_device(); s != EE_OK) return s;
  EE_CUDA(launch_peer_barrier((int* const*)signals->ptr, signals->rank, signals->world, epoch,
                              (DevStatus*)workspace, (cudaStream_t)stream));
  return EE_OK;
}

static CUresult (*get_addr_range())(CUdeviceptr*, size_t*, CUdeviceptr) {
  static CUresult (*fn)(CUdeviceptr*, size_t*, CUdeviceptr) = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) ==
            cudaSuccess && q == cudaDriverEntryPointSuccess)
      fn = (CUresult(*)(CUdeviceptr*, size_t*, CUdeviceptr))p;
  }
  return fn;
}

ee_status ee_ipc_get_handle(const void* dev_ptr, void* handle64, uint64_t* offset) {
  if (!dev_ptr || !handle64 || !offset) return fail(EE_ERR_ARG, "NULL argument");
  auto range = get_addr_range();
  if (!range) return fail(EE_ERR_CUDA, "cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, (CUdeviceptr)dev_ptr) != CUDA_SUCCESS)
    return fail(EE_ERR_CUDA, "cuMemGetAddressRange failed (not device memory?)");
  cudaIpcMemHandle_t h;
  EE_CUDA(cudaIpcGetMemHandle(&h, (void*)base));
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  memcpy(handle64, &h, sizeof(h));
  *offset = (uint64_t)((CUdeviceptr)dev_ptr - base);
  return EE_OK;
}

ee_status ee_ipc_open(const void* handle64, uint64_t offset, void** dev_ptr) {
  if (!handle64 || !dev_ptr) return fail(EE_ERR_ARG, "NULL argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof(h));
  void* base = nullptr;
  EE_CUDA(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
  *dev_ptr = (char*)base + offset;
  return EE_OK;
}

ee_status ee_ipc_close(void* dev_ptr, uint64_t offset) {
  if (!dev_ptr) return fail(EE_ERR_ARG, "NULL argument");
  EE_CUDA(cudaIpcCloseMemHandle((char*)dev_ptr - offset));
  return EE_OK;
}

ee_status ee_normalize_exit(const ee_head_config* cfg, ee_head_tensors* grads, float* loss,
                            const float* weight_sum, void* stream) {
  ee_status s = check_cfg(cfg);
  if (s != EE_OK) return s;
  if ((!grads && !loss) || !weight_sum) return fail(EE_ERR_ARG, "grads+loss/weight_sum NULL");
  if (grads && (s = check_arch_tensors(cfg, *grads, "grads", 0)) != EE_OK) return s;
  if ((s = check_device()) != EE_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  for (int k = 0; k < NTENS && grads; ++k) {
    float* g = (float*)(grads->*(kTens[k].f));
    if (!g) continue;
    Prof p_("normalize_exit", st, 0, 0, 8.0 * tensor_numel(cfg, k));
    EE_CUDA(launch_scale_by_inv(g, tensor_numel(cfg, k), weight_sum, st));
  }
  if (loss) EE_CUDA(launch_scale_by_inv(loss, 1, weight_sum, st));
  return EE_OK;
}

ee_status ee_init_heads(const ee_head_config* cfg, int32_t init, const ee_head_tensors* src,
                        int32_t src_dtype, uint64_t seed, float stdv, ee_head_tensors* master,
                        ee_head_tensors* op, void* stream) {
  ee_status s = check_cfg(cfg);
  if (s != EE_OK) return s;
  if (!master || !op) return fail(EE_ERR_ARG, "master/operand NULL");
  if (init != EE_INIT_COPY && init != EE_INIT_RANDOM) return fail(EE_ERR_ARG, "unknown init");
  if (src_dtype != EE_DTYPE_BF16 && src_dtype != EE_DTYPE_F32)
    return fail(EE_ERR_ARG, "unknown src_dtype");
  if (init == EE_INIT_COPY && !src) return fail(EE_ERR_STRUCTURE, "Copy init without a source");
  if ((s = check_device()) != EE_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  for (int i = 0; i < cfg->num_exits; ++i) {
    if ((s = check_arch_tensors(cfg, master[i], "master", i)) != EE_OK) return s;
    if ((s = check_arch_tensors(cfg, op[i], "operand", i)) != EE_OK) return s;
    for (int k = 0; k < NTENS; ++k) {
      const TInfo& ti = kTens[k];
      float* m = (float*)(master[i].*(ti.f));
      void* o = op[i].*(ti.f);
      const void* sp = src ? src[i].*(ti.f) : nullptr;
      if (!m) continue;
      const long long nel = tensor_numel(cfg, k);
      float* op_f32 = (ti.gain && o != (void*)m) ? (float*)o : nullptr;
      __nv_bfloat16* op_bf = ti.gain ? nullptr : (__nv_bfloat16*)o;
      if (init == EE_INIT_COPY) {
        if (!sp)
          return fail(EE_ERR_STRUCTURE, "Copy init: source module %s of exit %d is missing",
                      ti.name, i);
        if (!aligned16(sp)) return fail(EE_ERR_ALIGN, "copy source not 16-byte aligned");
        Prof p_("a0_init_copy", st, 0, 0, 8.0 * nel);
        EE_CUDA(launch_copy_cast(sp, src_dtype == EE_DTYPE_F32, m, op_bf, op_f32, nel, st));
      } else if (ti.gain) {
        Prof p_("a0_init_fill", st, 0, 0, 8.0 * nel);
        EE_CUDA(launch_fill(m, op_f32, nel, 1.0f, st));
      } else {
        Prof p_("a0_init_random", st, 0, 0, 6.0 * nel);
        EE_CUDA(launch_random_normal(seed, (uint64_t)i * 16 + k, stdv, m, op_bf, nel, st));
      }
    }
  }
  return EE_OK;
}

static ee_status opt_common(const ee_head_config* cfg, ee_head_tensors* master,
                            ee_head_tensors* op, const ee_head_tensors* grads) {
  ee_status s = check_cfg(cfg);
  if (s != EE_OK) return s;
  if (!master || !op || !grads) return fail(EE_ERR_ARG, "NULL argument");
  for (int i = 0; i < cfg->num_exits; ++i) {
    if ((s = check_arch_tensors(cfg, master[i], "master", i)) != EE_OK) return s;
    if ((s = check_arch_tensors(cfg, op[i], "operand", i)) != EE_OK) return s;
    if ((s = check_arch_tensors(cfg, grads[i], "grads", i)) != EE_OK) return s;
  }
  return check_device();
}

ee_status ee_adam_update(const ee_head_config* cfg, ee_head_tensors* master, ee_head_tensors* op,
                         const ee_head_tensors* grads, ee_head_tensors* m, ee_head_tensors* v,
                         float lr, float beta1, float beta2, float eps, float wd, int64_t step,
                         float grad_scale, void* stream) {
  ee_status s = opt_common(cfg, master, op, grads);
  if (s != EE_OK) return s;
  if (!m || !v) return fail(EE_ERR_ARG, "moments NULL");
  if (step < 1) return fail(EE_ERR_ARG, "step must be >= 1");
  cudaStream_t st = (cudaStream_t)stream;
  const float bc1 = (float)(1.0 - std::pow((double)beta1, (double)step));
  const float bc2 = (float)(1.0 - std::pow((double)beta2, (double)step));
  for (int i = 0; i < cfg->num_exits; ++i) {
    if ((s = check_arch_tensors(cfg, m[i], "m", i)) != EE_OK) return s;
    if ((s = check_arch_tensors(cfg, v[i], "v", i)) != EE_OK) return s;
    for (int k = 0; k < NTENS; ++k) {
      const TInfo& ti = kTens[k];
      float* mp = (float*)(master[i].*(ti.f));
      if (!mp) continue;
      void* opp = op[i].*(ti.f);
      float* opf = (ti.gain && opp != (void*)mp) ? (float*)opp : nullptr;
      __nv_bfloat16* opb = ti.gain ? nullptr : (__nv_bfloat16*)opp;
      const long long nel = tensor_numel(cfg, k);
      Prof p_("a15_adam", st, 0, 0, 30.0 * nel);
      EE_CUDA(launch_adam(mp, opb, opf, (const float*)(grads[i].*(ti.f)), (float*)(m[i].*(ti.f)),
                          (float*)(v[i].*(ti.f)), nel, lr, beta1, beta2, eps, wd, bc1, bc2,
                          grad_scale, st));
    }
  }
  return EE_OK;
}

ee_status ee_adam_update_sharded(const ee_head_config* cfg, int32_t world, int32_t rank,
                                const void* const* grad_arenas, ee_head_tensors* master_shard,
                                ee_head_tensors* m_shard, ee_head_tensors* v_shard,
                                const ee_peer_set* operands, float lr, float beta1, float beta2,
                                float eps, float wd, int64_t step, float grad_scale,
                                uint32_t tensor_mask, const float* grad_divisor,
                                void* stream) {
  ee_status s = check_cfg(cfg);
  if (s != EE_OK) return s;
  if (world < 1 || world > EE_MAX_PEERS || rank < 0 || rank >= world || !grad_arenas ||
      !master_shard || !m_shard || !v_shard || !operands)
    return fail(EE_ERR_ARG, "bad ee_adam_update_sharded arguments");
  if (step < 1) return fail(EE_ERR_ARG, "step must be >= 1");
  if ((s = check_device()) != EE_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  const float bc1 = (float)(1.0 - std::pow((double)beta1, (double)step));
  const float bc2 = (float)(1.0 - std::pow((double)beta2, (double)step));
  for (int i = 0; i < cfg->num_exits; ++i) {
    if (!grad_arenas[i] || !aligned16(grad_arenas[i]))
      return fail(EE_ERR_ALIGN, "grad_arenas[%d] NULL or misaligned", i);
    for (int k = 0; k < NTENS; ++k) {
      if (!in_arena(cfg, k)) continue;   // (a vocab shard's W_out has no arena block)
      if (tensor_mask && !(tensor_mask & (1u << k))) continue;
      long long R, C;
      tensor_rc(cfg, k, &R, &C);
      const long long rows = shard_rows(R, world, rank);
      if (rows == 0) continue;
      const TInfo& ti = kTens[k];
      float* th = (float*)(master_shard[i].*(ti.f));
      float* mm = (float*)(m_shard[i].*(ti.f));
      float* vv = (float*)(v_shard[i].*(ti.f));
      const ee_peer_set& op = operands[i * NTENS + k];
      if (!th || !mm || !vv || !aligned16(th) || !aligned16(mm) || !aligned16(vv))
        return fail(EE_ERR_ARG, "exit %d %s: shard tensors NULL or misaligned", i, ti.name);
      if (op.world != world || op.rank != rank)
        return fail(EE_ERR_ARG, "exit %d %s: operand peer set has wrong rank/world", i, ti.name);
      OpPeers pp{};
      pp.n = world;
      pp.f32 = ti.gain ? 1 : 0;
      for (int q = 0; q < world; ++q) {
        if (!op.ptr[q] || !aligned16(op.ptr[q]))
          return fail(EE_ERR_ALIGN, "exit %d %s: operand %d NULL or misaligned", i, ti.name, q);
        pp.p[q] = op.ptr[q];
      }
      const float* slots = (const float*)grad_arenas[i] + arena_offset(cfg, world, rank, k);
      const long long nel = rows * C;
      Prof p_("a15_adam_sharded", st, 0, 0, (4.0 * world + 24.0 + 2.0 * world) * nel);
      EE_CUDA(launch_adam_sharded(th, slots, world, mm, vv, nel, pp,
                                  (long long)rank * shard_chunk(R, world) * C, lr, beta1, beta2,
                                  eps, wd, bc1, bc2, grad_scale, st,
                                  grad_divisor ? grad_divisor + i : nullptr));
    }
  }
  return EE_OK;
}

ee_status ee_sgd_update(const ee_head_config* cfg, ee_head_tensors* master, ee_head_tensors* op,
                        const ee_head_tensors* grads, ee_head_tensors* buf, float lr,
                        float momentum, float grad_scale, void* stream) {
  ee_status s = opt_common(cfg, master, op, grads);
  if (s != EE_OK) return s;
  if (momentum != 0.f && !buf) return fail(EE_ERR_ARG, "momentum buffer required");
  cudaStream_t st = (cudaStream_t)stream;
  for (int i = 0; i < cfg->num_exits; ++i) {
    for (int k = 0; k < NTENS; ++k) {
      const TInfo& ti = kTens[k];
      float* mp = (float*)(master[i].*(ti.f));
      if (!mp) continue;
      void* opp = op[i].*(ti.f);
      float* opf = (ti.gain && opp != (void*)mp) ? (float*)opp : nullptr;
      __nv_bfloat16* opb = ti.gain ? nullptr : (__nv_bfloat16*)opp;
      float* bk = (buf && momentum != 0.f) ? (float*)(buf[i].*(ti.f)) : nullptr;
      const long long nel = tensor_numel(cfg, k);
      Prof p_("a15_sgd", st, 0, 0, 14.0 * nel);
      EE_CUDA(launch_sgd(mp, opb, opf, (const float*)(grads[i].*(ti.f)), bk, nel, lr, momentum,
                         grad_scale, st));
    }
  }
  return EE_OK;
}


ee_status ee_profile_start(void) {
  for (auto& r : g_prof) {
    g_event_pool.push_back(r.a);
    g_event_pool.push_back(r.b);
  }
  g_prof.clear();
  g_prof_on = true;
  return EE_OK;
}

ee_status ee_profile_stop(int32_t* count) {
  g_prof_on = false;
  if (count) *count = (int32_t)g_prof.size();
  return EE_OK;
}

ee_status ee_profile_record(int32_t i, char* name, int32_t name_len, float* ms, double* flops_exec,
                            double* flops_alg, double* bytes) {
  if (i < 0 || i >= (int32_t)g_prof.size()) return fail(EE_ERR_ARG, "profile index out of range");
  const ProfRec& r = g_prof[i];
  EE_CUDA(cudaEventSynchronize(r.b));
  float t = 0.f;
  EE_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
  if (name && name_len > 0) {
    strncpy(name, r.name, name_len - 1);
    name[name_len - 1] = 0;
  }
  if (ms) *ms = t;
  if (flops_exec) *flops_exec = r.flops_exec;
  if (flops_alg) *flops_alg = r.flops_alg;
  if (bytes) *bytes = r.bytes;
  return EE_OK;
}

int64_t ee_launch_count(void) { return g_launches.load(); }

// Debug hook (not in ee.h's product surface): arm a per-tile timing trace of the
// next GEMM launch, then read (globaltimer_ns << 8 | smid) per tile.
void ee_debug_trace_arm(void) { debug_trace_arm(); }
int32_t ee_debug_trace_read(uint64_t* host, int32_t max) {
  cudaDeviceSynchronize();
  return debug_trace_read((unsigned long long*)host, max);
}

// Testing hook: causal GQA attention forward (o, lse2) and backward (dq, dk, dv)
// on q [N x Hq*128], k, v [N x Hkv*128] bf16 (RoPE not applied).  dout may be
// NULL (forward only).  scratch: fp32 [N*Hq] for rowsum(dO*O).
ee_status ee_test_attention(const void* q, const void* k, const void* v, void* o, float* lse2,
                            const void* dout, void* dq, void* dk, void* dv, float* scratch,
                            int64_t n_tokens, int32_t seq_len, int32_t n_heads, int32_t n_kv_heads,
                            int32_t impl, void* stream) {
  if (!q || !k || !v || !o || !lse2 || n_tokens < 0 || seq_len < 64 || seq_len % 64 ||
      n_tokens % seq_len || n_heads < 1 || n_kv_heads < 1 || n_heads % n_kv_heads)
    return fail(EE_ERR_ARG, "bad ee_test_attention arguments");
  ee_status s = check_device();
  if (s != EE_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  if (impl < 0 || impl > 2) return fail(EE_ERR_ARG, "impl must be 0, 1 or 2");
  EE_CUDA(attn_forward_impl(impl, (const __nv_bfloat16*)q, (const __nv_bfloat16*)k,
                            (const __nv_bfloat16*)v, (__nv_bfloat16*)o, n_tokens, seq_len,
                            n_heads, n_kv_heads, lse2, st));
  if (dout) {
    if (!dq || !dk || !dv || !scratch) return fail(EE_ERR_ARG, "backward outputs NULL");
    EE_CUDA(launch_attn_bwd((const __nv_bfloat16*)q, (const __nv_bfloat16*)k,
                            (const __nv_bfloat16*)v, (const __nv_bfloat16*)o,
                            (const __nv_bfloat16*)dout, lse2, scratch, (__nv_bfloat16*)dq,
                            (__nv_bfloat16*)dk, (__nv_bfloat16*)dv, n_tokens, seq_len, n_heads,
                            n_kv_heads, 0.f, st, impl != 0));
  }
  return EE_OK;
}

// Testing hook: C[M x N] (fp32, row-major) (+)= A B^T with A stored [M x K]
// (a_kmajor) or [K x M], B stored [N x K] (b_kmajor) or [K x N]; bf16.
ee_status ee_test_gemm(int32_t a_kmajor, int32_t b_kmajor, const void* A, const void* B, float* C,
                       int32_t M, int32_t N, int32_t K, int32_t accumulate, void* stream) {
  if (!A || !B || !C || M < 1 || N < 1 || K < 1) return fail(EE_ERR_ARG, "bad test_gemm args");
  if (K % 8 || (!a_kmajor && M % 8) || (!b_kmajor && N % 8) || N % 4)
    return fail(EE_ERR_SHAPE, "test_gemm: strides must be 16-byte multiples");
  ee_status s = check_device();
  if (s != EE_OK) return s;
  GemmArgs a = base_args(M, N, K);
  a.out0 = C;
  a.ldo = N;
  a.accumulate = accumulate;
  Mat mA = a_kmajor ? Mat{A, M, K, K} : Mat{A, K, M, M};
  Mat mB = b_kmajor ? Mat{B, N, K, K} : Mat{B, K, N, N};
  EE_CUDA(gemm_run(EPI_F32, a_kmajor != 0, b_kmajor != 0, mA, mB, nullptr, B_PLAIN, 0, a,
                   (cudaStream_t)stream));
  return EE_OK;
}

}  // extern "C"
