// comm.cu -- the in-library communicator (include/ee.h ee_comm_*): one
// ee_tune_step call runs a data-parallel or vocab-parallel step over the
// ranks of a node, with every exchange done by this library's kernels over
// NVLink peer memory (CUDA IPC mappings of each rank's symmetric arena).
//
// PAPER.md §2.2 "Support for 3D parallelism": EE-Tuning runs
// under data and tensor/vocabulary parallelism because the exits are
// independent and the loss is a sum over independent tokens
// (P:183-188).  The step is composed from the library's own entry points
// (ee_tune_step_rs, ee_vp_*, ee_peer_barrier) plus the small kernels below:
//   - rank-ordered reductions of small vectors (valid count, losses, CE
//     statistics) read from every rank's arena (deterministic: fixed order);
//   - the owner-side sum of the gradient slots a peer's GEMM epilogue stored
//     (the fused reduce-scatter's second half), and the all-gather of the
//     reduced rows into every rank's gradient tensors (peer loads).
// No NCCL and no host synchronisation: everything is stream-ordered, and
// ranks are ordered against each other by ee_peer_barrier.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <cstdint>
#include <cstring>
#include <new>
#include "../../include/ee.h"

namespace ee {
ee_status comm_fail(ee_status s, const char* msg);   // api.cu: sets ee_last_error()
}

struct ee_comm {
  int32_t mode, world, rank;
  ee_head_config cfg;          // shapes the arena was sized for (num_exits = 1)
  int64_t n_local;
  char* arena[EE_MAX_PEERS];   // every rank's arena, mapped into this process
  size_t bytes;
  size_t off_sig, off_small, off_tg, off_z, off_key, off_sums, off_keyg, off_sumsg, off_slots;
  size_t off_grad[2];
  uint32_t epoch;
};

namespace {

using ee::comm_fail;

constexpr int NT = 11;         // ee_head_tensors members, in order
void* ee_head_tensors::*const kMember[NT] = {
    &ee_head_tensors::g_a,  &ee_head_tensors::w_gate, &ee_head_tensors::w_up,
    &ee_head_tensors::w_down, &ee_head_tensors::g_f,  &ee_head_tensors::w_out,
    &ee_head_tensors::g_att, &ee_head_tensors::w_q,   &ee_head_tensors::w_k,
    &ee_head_tensors::w_v,  &ee_head_tensors::w_o};
constexpr int MAXE = 64;       // exits per call (small-region slots)

#define COMM_CUDA(call)                                                            \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess) return comm_fail(EE_ERR_CUDA, cudaGetErrorString(e_));  \
  } while (0)
#define COMM_TRY(call)                   \
  do {                                   \
    ee_status s_ = (call);               \
    if (s_ != EE_OK) return s_;          \
  } while (0)

size_t up(size_t x) { return (x + 255) & ~(size_t)255; }

// Small region (bytes): [0] int64 local valid count, [8] int64 global count,
// [64] float loss[MAXE], [64 + 4 MAXE] float wsum[MAXE],
// [64 + 8 MAXE] float loss_g[MAXE], [64 + 12 MAXE] float wsum_g[MAXE].
constexpr size_t SM_CNT = 0, SM_CNTG = 8, SM_LOSS = 64, SM_WSUM = 64 + 4 * MAXE,
                 SM_LOSSG = 64 + 8 * MAXE, SM_WSUMG = 64 + 12 * MAXE,
                 SM_BYTES = 64 + 16 * MAXE;

// Largest arena of the fused gradient reduce-scatter over the ranks (the
// last rank's row shards can be shorter; size every arena for the largest).
ee_status grad_arena_floats(const ee_head_config* c1, int world, long long* out) {
  long long best = 0;
  for (int q = 0; q < world; ++q) {
    int64_t rb, rows, off, tot;
    COMM_TRY(ee_dp_shard_layout(c1, world, q, 0, &rb, &rows, &off, &tot));
    if (tot > best) best = tot;
  }
  *out = best;
  return EE_OK;
}

ee_status layout(const ee_head_config* cfg, int mode, int world, int64_t n_local, ee_comm* L) {
  ee_head_config c1 = *cfg;
  c1.num_exits = 1;
  const size_t h = (size_t)cfg->hidden, n_all = (size_t)world * (size_t)n_local;
  size_t o = 0;
  L->off_sig = o;   o += up(sizeof(int32_t) * EE_MAX_PEERS);
  L->off_small = o; o += up(SM_BYTES);
  L->off_tg = L->off_z = L->off_key = L->off_sums = L->off_keyg = L->off_sumsg = L->off_slots = 0;
  if (mode == EE_COMM_VP) {
    L->off_tg = o;    o += up(4 * n_all);
    L->off_z = o;     o += up(2 * n_all * h);
    L->off_key = o;   o += up(8 * n_all);
    L->off_sums = o;  o += up(8 * n_all);
    L->off_keyg = o;  o += up(8 * n_all);
    L->off_sumsg = o; o += up(8 * n_all);
    if (cfg->arch != EE_ARCH_EMBEDDING) {
      L->off_slots = o;
      o += up(4 * (size_t)world * (size_t)n_local * h);
    }
  }
  long long gf = 0;
  const bool grads = mode == EE_COMM_DP || cfg->arch != EE_ARCH_EMBEDDING;
  if (grads) COMM_TRY(grad_arena_floats(&c1, world, &gf));
  for (int j = 0; j < 2; ++j) {
    L->off_grad[j] = o;
    o += up(4 * (size_t)gf);
  }
  L->bytes = o;
  return EE_OK;
}

// ---------------------------------------------------------------- kernels
struct Srcs {
  const void* p[EE_MAX_PEERS];
};

// out[j] = src_0[j] (+|max) src_1[j] ... in rank order (deterministic).
template <typename T, bool MAX>
__global__ void peer_reduce_kernel(Srcs s, int P, long long n, T* __restrict__ out) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n;
       j += (long long)gridDim.x * blockDim.x) {
    T a = ((const T*)s.p[0])[j];
    for (int q = 1; q < P; ++q) {
      const T b = ((const volatile T*)s.p[q])[j];
      a = MAX ? (b > a ? b : a) : a + b;
    }
    out[j] = a;
  }
}

// The owner's sum of one tensor's gradient slots: block [P][len] -> slot 0
// = sum over q in rank order (the same order ee_adam_update_sharded uses).
__global__ void slot_sum_kernel(float4* __restrict__ block, int P, long long len4) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < len4;
       j += (long long)gridDim.x * blockDim.x) {
    float4 a = block[j];
    for (int q = 1; q < P; ++q) {
      const float4 b = block[q * len4 + j];
      a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
    }
    block[j] = a;
  }
}

// All-gather of the reduced rows: for owner q = blockIdx.y, copy (or add)
// n4[q] float4s from its reduced slot (peer memory) to dst + dst_off4[q].
struct Gather {
  const float4* src[EE_MAX_PEERS];
  long long dst_off4[EE_MAX_PEERS];
  long long n4[EE_MAX_PEERS];
};
__global__ void gather_kernel(Gather g, float4* __restrict__ dst, int accumulate) {
  const int q = blockIdx.y;
  const long long n4 = g.n4[q];
  const float4* __restrict__ src = g.src[q];
  float4* d = dst + g.dst_off4[q];
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n4;
       j += (long long)gridDim.x * blockDim.x) {
    float4 v = src[j];
    if (accumulate) {
      const float4 o = d[j];
      v.x += o.x; v.y += o.y; v.z += o.z; v.w += o.w;
    }
    d[j] = v;
  }
}

int grid_for(long long n, int threads, int cap) {
  long long b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  return (int)(b < cap ? b : cap);
}

template <typename T, bool MAX>
ee_status peer_reduce(const ee_comm* c, size_t off, long long n, T* out, cudaStream_t st) {
  if (n <= 0) return EE_OK;
  Srcs s{};
  for (int q = 0; q < c->world; ++q) s.p[q] = c->arena[q] + off;
  peer_reduce_kernel<T, MAX><<<grid_for(n, 256, 4 * 148), 256, 0, st>>>(s, c->world, n, out);
  COMM_CUDA(cudaGetLastError());
  return EE_OK;
}

ee_status barrier(ee_comm* c, void* ws, cudaStream_t st) {
  nvtxRangePushA("ee_comm barrier");
  struct Pop { ~Pop() { nvtxRangePop(); } } pop_;
  ee_peer_set sig;
  memset(&sig, 0, sizeof(sig));
  sig.rank = c->rank;
  sig.world = c->world;
  for (int q = 0; q < c->world; ++q) sig.ptr[q] = c->arena[q] + c->off_sig;
  return ee_peer_barrier(&sig, ++c->epoch, ws, st);
}

ee_peer_set pset(const ee_comm* c, size_t off) {
  ee_peer_set p;
  memset(&p, 0, sizeof(p));
  p.rank = c->rank;
  p.world = c->world;
  for (int q = 0; q < c->world; ++q) p.ptr[q] = c->arena[q] + off;
  return p;
}

// Owner-side sum of arena j's slots, then every rank gathers the reduced rows
// of every owner into grads (the all-reduce's second half).  Two barriers:
// all partials landed before the sum, all sums done before the gather.
ee_status reduce_gather(ee_comm* c, const ee_head_config* c1, int j, ee_head_tensors* grads,
                        int accumulate, void* ws, cudaStream_t st) {
  const int P = c->world;
  nvtxRangePushA("ee_comm gradient reduce + gather");
  struct Pop { ~Pop() { nvtxRangePop(); } } pop_;
  COMM_TRY(barrier(c, ws, st));
  float* own = (float*)(c->arena[c->rank] + c->off_grad[j]);
  for (int k = 0; k < NT; ++k) {
    int64_t rb, rows, off, tot;
    COMM_TRY(ee_dp_shard_layout(c1, P, c->rank, k, &rb, &rows, &off, &tot));
    int64_t rb1, rows1, off1, tot1;    // next block's offset = this block's end
    COMM_TRY(ee_dp_shard_layout(c1, P, c->rank, k + 1 < NT ? k + 1 : k, &rb1, &rows1, &off1,
                                &tot1));
    const long long end = k + 1 < NT ? off1 : tot;
    if (end == off || rows == 0) continue;            // not in the arena / no rows owned
    const long long len = (end - off) / P;            // rows * C
    slot_sum_kernel<<<grid_for(len / 4, 256, 8 * 148), 256, 0, st>>>((float4*)(own + off), P,
                                                                      len / 4);
    COMM_CUDA(cudaGetLastError());
  }
  COMM_TRY(barrier(c, ws, st));
  for (int k = 0; k < NT; ++k) {
    float* dst = (float*)(grads->*kMember[k]);
    Gather g;
    memset(&g, 0, sizeof(g));
    long long most = 0;
    bool any = false;
    for (int q = 0; q < P; ++q) {
      int64_t rb, rows, off, tot, rb1, rows1, off1, tot1;
      COMM_TRY(ee_dp_shard_layout(c1, P, q, k, &rb, &rows, &off, &tot));
      COMM_TRY(ee_dp_shard_layout(c1, P, q, k + 1 < NT ? k + 1 : k, &rb1, &rows1, &off1, &tot1));
      const long long end = k + 1 < NT ? off1 : tot;
      if (end == off) continue;                       // tensor not reduced through the arena
      any = true;
      const long long len = (end - off) / P;
      g.src[q] = (const float4*)((const float*)(c->arena[q] + c->off_grad[j]) + off);
      g.dst_off4[q] = len ? (rb * (len / (rows ? rows : 1))) / 4 : 0;
      g.n4[q] = len / 4;
      if (g.n4[q] > most) most = g.n4[q];
    }
    if (!any) continue;
    if (!dst) return comm_fail(EE_ERR_ARCH, "ee_tune_step(comm): a gradient tensor is NULL");
    dim3 grid(grid_for(most, 256, 2 * 148), P);
    gather_kernel<<<grid, 256, 0, st>>>(g, (float4*)dst, accumulate);
    COMM_CUDA(cudaGetLastError());
  }
  return EE_OK;
}

ee_status dp_step(ee_comm* c, const ee_head_config* cfg, const void* const* hidden,
                  int64_t n_local, const int32_t* targets, const float* exit_weights,
                  const ee_head_tensors* params, ee_head_tensors* grads, int32_t accumulate,
                  float* loss_out, const ee_step_aux* aux, const int64_t* valid_count, void* ws,
                  size_t ws_bytes, cudaStream_t st) {
  const int E = cfg->num_exits;
  const bool conf = cfg->token_weighting == EE_WEIGHT_CONFIDENCE;
  ee_head_config c1 = *cfg;
  c1.num_exits = 1;
  if (conf) c1.token_weighting = EE_WEIGHT_CONFIDENCE_SUM;
  char* sm = c->arena[c->rank] + c->off_small;
  const int64_t* W = valid_count;
  if (!conf && !W) {   // global valid-token count: local counts summed in rank order
    COMM_TRY(ee_count_valid(targets, n_local, cfg->vocab, (int64_t*)(sm + SM_CNT), ws, ws_bytes,
                            st));
    COMM_TRY(barrier(c, ws, st));
    COMM_TRY((peer_reduce<long long, false>(c, c->off_small + SM_CNT, 1,
                                            (long long*)(sm + SM_CNTG), st)));
    W = (const int64_t*)(sm + SM_CNTG);
  }
  if (conf) W = nullptr;
  for (int i = 0; i < E; ++i) {
    const int j = i & 1;
    ee_peer_set ar = pset(c, c->off_grad[j]);
    ee_step_aux ax;
    memset(&ax, 0, sizeof(ax));
    if (aux) ax = aux[i];
    if (conf) ax.weight_sum = (float*)(sm + SM_WSUM) + i;
    COMM_TRY(ee_tune_step_rs(&c1, &hidden[i], n_local, targets, &exit_weights[i], &params[i], &ar,
                             (float*)(sm + SM_LOSS) + i, &ax, W, ws, ws_bytes, st));
    COMM_TRY(reduce_gather(c, &c1, j, &grads[i], accumulate, ws, st));
  }
  // losses (and confidence weight sums) summed over the ranks in rank order
  COMM_TRY(barrier(c, ws, st));
  COMM_TRY((peer_reduce<float, false>(c, c->off_small + SM_LOSS, E, (float*)(sm + SM_LOSSG), st)));
  if (conf) {
    COMM_TRY((peer_reduce<float, false>(c, c->off_small + SM_WSUM, E, (float*)(sm + SM_WSUMG),
                                        st)));
    for (int i = 0; i < E; ++i)   // L_i = sum c_t loss_t / sum c_t over all ranks (A17)
      COMM_TRY(ee_normalize_exit(&c1, &grads[i], (float*)(sm + SM_LOSSG) + i,
                                 (const float*)(sm + SM_WSUMG) + i, st));
  }
  COMM_CUDA(cudaMemcpyAsync(loss_out, sm + SM_LOSSG, sizeof(float) * E, cudaMemcpyDeviceToDevice,
                            st));
  if (conf && aux)
    for (int i = 0; i < E; ++i)
      if (aux[i].weight_sum)
        COMM_CUDA(cudaMemcpyAsync(aux[i].weight_sum, (float*)(sm + SM_WSUMG) + i, sizeof(float),
                                  cudaMemcpyDeviceToDevice, st));
  return EE_OK;
}

ee_status vp_step(ee_comm* c, const ee_head_config* cfg, const void* const* hidden,
                  int64_t n_local, const int32_t* targets, const float* exit_weights,
                  const ee_head_tensors* params, ee_head_tensors* grads, int32_t accumulate,
                  float* loss_out, const ee_step_aux* aux, const int64_t* valid_count, void* ws,
                  size_t ws_bytes, cudaStream_t st) {
  const int E = cfg->num_exits, P = c->world;
  const int64_t n_all = (int64_t)P * n_local;
  ee_head_config c1 = *cfg;
  c1.num_exits = 1;
  char* mine = c->arena[c->rank];
  char* sm = mine + c->off_small;
  // targets all-gather: this rank's ids into every rank's targets_all
  for (int q = 0; q < P; ++q)
    COMM_CUDA(cudaMemcpyAsync(c->arena[q] + c->off_tg + 4 * (size_t)c->rank * n_local, targets,
                              4 * (size_t)n_local, cudaMemcpyDeviceToDevice, st));
  COMM_TRY(barrier(c, ws, st));
  const int32_t* tg_all = (const int32_t*)(mine + c->off_tg);
  const int64_t* W = valid_count;
  if (!W) {
    COMM_TRY(ee_count_valid(tg_all, n_all, cfg->vocab, (int64_t*)(sm + SM_CNTG), ws, ws_bytes,
                            st));
    W = (const int64_t*)(sm + SM_CNTG);
  }
  const bool body = cfg->arch != EE_ARCH_EMBEDDING;
  ee_peer_set zset = pset(c, c->off_z), slots = pset(c, c->off_slots);
  int64_t* key = (int64_t*)(mine + c->off_key);
  float* sums = (float*)(mine + c->off_sums);
  int64_t* keyg = (int64_t*)(mine + c->off_keyg);
  float* sumsg = (float*)(mine + c->off_sumsg);
  const void* z_all = mine + c->off_z;
  for (int i = 0; i < E; ++i) {
    COMM_TRY(ee_vp_exit_forward_ag(&c1, hidden[i], n_local, n_all, &params[i], &zset, ws,
                                   ws_bytes, st));                                  // a1-a4 + AG
    COMM_TRY(barrier(c, ws, st));
    COMM_TRY(ee_vp_vocab_stats(&c1, z_all, n_all, tg_all, &params[i], key, sums, ws, ws_bytes,
                               st));                                                // a5
    COMM_TRY(barrier(c, ws, st));
    COMM_TRY((peer_reduce<long long, true>(c, c->off_key, n_all, (long long*)keyg, st)));
    COMM_TRY(ee_vp_rescale(&c1, n_all, keyg, sums, ws, ws_bytes, st));
    COMM_TRY(barrier(c, ws, st));
    COMM_TRY((peer_reduce<float, false>(c, c->off_sums, 2 * n_all, sumsg, st)));
    const ee_step_aux* ax = aux ? &aux[i] : nullptr;
    if (body)
      COMM_TRY(ee_vp_vocab_backward_rs(&c1, z_all, n_all, tg_all, keyg, sumsg, exit_weights[i], W,
                                       &params[i], &grads[i], accumulate, &slots, loss_out + i,
                                       ax, i, ws, ws_bytes, st));                   // a6-a9 + RS
    else
      COMM_TRY(ee_vp_vocab_backward(&c1, z_all, n_all, tg_all, keyg, sumsg, exit_weights[i], W,
                                    &params[i], &grads[i], accumulate, nullptr, loss_out + i, ax,
                                    i, ws, ws_bytes, st));
    COMM_TRY(barrier(c, ws, st));
    if (!body) continue;
    const int j = i & 1;
    ee_peer_set ar = pset(c, c->off_grad[j]);
    COMM_TRY(ee_vp_exit_backward_slots(&c1, hidden[i], n_local, n_all, &params[i],
                                       (const float*)(mine + c->off_slots), P, &grads[i], 0, &ar,
                                       ws, ws_bytes, st));                          // a10-a13
    COMM_TRY(reduce_gather(c, &c1, j, &grads[i], accumulate, ws, st));
  }
  return EE_OK;
}

}  // namespace

namespace ee {
// Called by ee_tune_step when comm != NULL (api.cu).
ee_status comm_tune_step(const ee_comm* cc, const ee_head_config* cfg, const void* const* hidden,
                         int64_t n_tokens, const int32_t* targets, const float* exit_weights,
                         const ee_head_tensors* params, ee_head_tensors* grads, int32_t accumulate,
                         float* loss_out, const ee_step_aux* aux, const int64_t* valid_count,
                         void* workspace, size_t ws_bytes, void* stream) {
  ee_comm* c = const_cast<ee_comm*>(cc);   // the barrier epoch advances
  const cudaStream_t st = (cudaStream_t)stream;
  if (!cfg || !hidden || !exit_weights || !params || !grads || !loss_out || n_tokens <= 0 ||
      !targets || !workspace)
    return comm_fail(EE_ERR_ARG, "ee_tune_step(comm): NULL argument or n_tokens <= 0");
  if (cfg->num_exits > MAXE) return comm_fail(EE_ERR_SHAPE, "ee_tune_step(comm): > 64 exits");
  if (n_tokens != c->n_local || cfg->hidden != c->cfg.hidden || cfg->vocab != c->cfg.vocab ||
      cfg->ffn != c->cfg.ffn || cfg->arch != c->cfg.arch ||
      cfg->vocab_begin != c->cfg.vocab_begin || cfg->vocab_end != c->cfg.vocab_end ||
      cfg->n_kv_heads != c->cfg.n_kv_heads)
    return comm_fail(EE_ERR_SHAPE, "ee_tune_step(comm): shapes differ from ee_comm_create's");
  if (c->mode == EE_COMM_DP)
    return dp_step(c, cfg, hidden, n_tokens, targets, exit_weights, params, grads, accumulate,
                   loss_out, aux, valid_count, workspace, ws_bytes, st);
  return vp_step(c, cfg, hidden, n_tokens, targets, exit_weights, params, grads, accumulate,
                 loss_out, aux, valid_count, workspace, ws_bytes, st);
}
}  // namespace ee

extern "C" {

ee_status ee_comm_arena_size(const ee_head_config* cfg, int32_t mode, int32_t world,
                             int64_t n_local, size_t* bytes) {
  if (!cfg || !bytes || n_local < 1 || world < 1 || world > EE_MAX_PEERS ||
      (mode != EE_COMM_DP && mode != EE_COMM_VP))
    return comm_fail(EE_ERR_ARG, "ee_comm_arena_size: bad arguments");
  size_t ws;
  COMM_TRY(ee_workspace_size(cfg, n_local, &ws));       // validates cfg
  ee_comm L;
  COMM_TRY(layout(cfg, mode, world, n_local, &L));
  *bytes = L.bytes;
  return EE_OK;
}

ee_status ee_comm_create(ee_comm** out, const ee_head_config* cfg, int32_t mode, int32_t world,
                         int32_t rank, int64_t n_local, void* const* arenas, size_t arena_bytes) {
  if (!out || !cfg || !arenas || world < 1 || world > EE_MAX_PEERS || rank < 0 ||
      rank >= world || n_local < 1 || (mode != EE_COMM_DP && mode != EE_COMM_VP))
    return comm_fail(EE_ERR_ARG, "ee_comm_create: bad arguments");
  if (mode == EE_COMM_VP) {
    if (cfg->vocab_end <= cfg->vocab_begin)
      return comm_fail(EE_ERR_ARG, "ee_comm_create(VP): empty vocab shard");
  } else if (cfg->vocab_begin != 0 || cfg->vocab_end != cfg->vocab) {
    return comm_fail(EE_ERR_ARG, "ee_comm_create(DP): W_out must be unsharded");
  }
  ee_comm* c = new (std::nothrow) ee_comm;
  if (!c) return comm_fail(EE_ERR_ARG, "ee_comm_create: out of host memory");
  memset(c, 0, sizeof(*c));
  ee_status s = layout(cfg, mode, world, n_local, c);
  if (s != EE_OK) {
    delete c;
    return s;
  }
  if (arena_bytes < c->bytes) {
    delete c;
    return comm_fail(EE_ERR_WORKSPACE, "ee_comm_create: arena smaller than ee_comm_arena_size");
  }
  for (int q = 0; q < world; ++q) {
    if (!arenas[q] || ((uintptr_t)arenas[q] & 255u)) {
      delete c;
      return comm_fail(EE_ERR_ALIGN, "ee_comm_create: arena pointer NULL or not 256-B aligned");
    }
    c->arena[q] = (char*)arenas[q];
  }
  c->mode = mode;
  c->world = world;
  c->rank = rank;
  c->cfg = *cfg;
  c->cfg.num_exits = 1;
  c->n_local = n_local;
  c->epoch = 0;
  *out = c;
  return EE_OK;
}

ee_status ee_comm_destroy(ee_comm* comm) {
  delete comm;
  return EE_OK;
}

}  // extern "C"
