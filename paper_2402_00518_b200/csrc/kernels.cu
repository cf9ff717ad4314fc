// kernels.cu -- the bandwidth-bound kernels of the exit-head step:
// RMSNorm forward/backward, gain gradients, cross-entropy
// finalisation (merge of the per-tile online-softmax partials),
// loss reduction, valid-token count, Adam/SGD and initialisers
// (P:227-238).  All reductions are deterministic (fixed order, no float
// atomics), so reruns are bitwise identical.
#include <algorithm>
#include <cfloat>
#include <climits>
#include <cuda_fp16.h>
#include "internal.cuh"

namespace ee {

// ---------------------------------------------------------------- helpers
__device__ __forceinline__ void load8(const __nv_bfloat16* p, float (&v)[8]) {
  const uint4 q = *reinterpret_cast<const uint4*>(p);
  const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    v[2 * i] = bf16lo(w[i]);
    v[2 * i + 1] = bf16hi(w[i]);
  }
}
__device__ __forceinline__ void load8(const float* p, float (&v)[8]) {
  const float4 a = *reinterpret_cast<const float4*>(p);
  const float4 b = *reinterpret_cast<const float4*>(p + 4);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
  v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ void store8(__nv_bfloat16* p, const float (&v)[8]) {
  uint4 q;
  q.x = pack_bf16(v[0], v[1]);
  q.y = pack_bf16(v[2], v[3]);
  q.z = pack_bf16(v[4], v[5]);
  q.w = pack_bf16(v[6], v[7]);
  *reinterpret_cast<uint4*>(p) = q;
}

// Block-wide sum (deterministic: fixed shuffle tree, then warp 0 over warps).
template <typename T>
__device__ __forceinline__ T block_sum(T v, T* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int nw = (blockDim.x + 31) >> 5;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    T t = l < nw ? red[l] : T(0);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (l == 0) red[32] = t;
  }
  __syncthreads();
  return red[32];
}

// Each thread owns up to 2 chunks of 8 consecutive columns: h <= 16*blockDim.
constexpr int NORM_CHUNKS = 2;
static inline int norm_threads(int h) {
  int t = (h / 8 + NORM_CHUNKS - 1) / NORM_CHUNKS;
  return ((t + 31) / 32) * 32;
}

// ---------------------------------------------------------------- valid count
__global__ void count_valid_kernel(const int32_t* __restrict__ y, long long n, int vocab,
                                   long long* out, DevStatus* st) {
  __shared__ long long red[33];
  long long c = 0;
  bool bad = false;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) {
    const int t = y[i];
    c += (t != -1);
    bad |= (t < -1 || t >= vocab);
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) set_status(st, 4 /*EE_ERR_VOCAB*/, -1);
  c = block_sum(c, red);
  if (threadIdx.x == 0) out[0] = c;
}

cudaError_t launch_count_valid(const int32_t* targets, long long n, int vocab, long long* out,
                               DevStatus* st, cudaStream_t s) {
  count_valid_kernel<<<1, 1024, 0, s>>>(targets, n, vocab, out, st);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- RMSNorm fwd
// out = g * x * r, r = rsqrt(mean x^2 + eps)   (A3)
template <typename TIn>
__global__ void rmsnorm_fwd_kernel(const TIn* __restrict__ in, const float* __restrict__ g,
                                   float eps, __nv_bfloat16* __restrict__ out,
                                   float* __restrict__ r, int h, PeerRows ag) {
  __shared__ float red[33];
  const long long row = blockIdx.x;
  const int nchunk = h / 8;
  griddep_launch();  // no-ops unless launched with PDL (the decode chain)
  griddep_wait();
  float x[NORM_CHUNKS][8];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < NORM_CHUNKS; ++i) {
    const int c = threadIdx.x + i * blockDim.x;
    if (c < nchunk) {
      load8(in + row * h + c * 8, x[i]);
#pragma unroll
      for (int k = 0; k < 8; ++k) ss += x[i][k] * x[i][k];
    }
  }
  ss = block_sum(ss, red);
  const float rr = 1.0f / sqrtf(ss / (float)h + eps);
#pragma unroll
  for (int i = 0; i < NORM_CHUNKS; ++i) {
    const int c = threadIdx.x + i * blockDim.x;
    if (c < nchunk) {
      float gv[8], o[8];
      load8(g + c * 8, gv);
#pragma unroll
      for (int k = 0; k < 8; ++k) o[k] = gv[k] * (x[i][k] * rr);
      if (ag.n == 0) {
        store8(out + row * h + c * 8, o);
      } else {  // fused all-gather: the same 16 bytes to every rank's z_all (NVLink stores)
#pragma unroll
        for (int q = 0; q < MAX_PEERS; ++q)  // constant indices: the table stays in param space
          if (q < ag.n) store8(ag.p[q] + (ag.row_off + row) * h + c * 8, o);
      }
    }
  }
  if (threadIdx.x == 0) r[row] = rr;
}

cudaError_t launch_rmsnorm_fwd(const void* in, bool in_f32, const float* g, float eps,
                               __nv_bfloat16* out, float* r, long long n, int h, cudaStream_t s,
                               const PeerRows* ag, bool pdl) {
  if (n == 0) return cudaSuccess;
  const int t = norm_threads(h);
  PeerRows pr{};
  if (ag) pr = *ag;
  if (pdl) {
    if (in_f32)
      return launch_pdl(rmsnorm_fwd_kernel<float>, dim3((unsigned)n), dim3(t), 0, s,
                        (const float*)in, g, eps, out, r, h, pr);
    return launch_pdl(rmsnorm_fwd_kernel<__nv_bfloat16>, dim3((unsigned)n), dim3(t), 0, s,
                      (const __nv_bfloat16*)in, g, eps, out, r, h, pr);
  }
  if (in_f32)
    rmsnorm_fwd_kernel<float><<<(unsigned)n, t, 0, s>>>((const float*)in, g, eps, out, r, h, pr);
  else
    rmsnorm_fwd_kernel<__nv_bfloat16>
        <<<(unsigned)n, t, 0, s>>>((const __nv_bfloat16*)in, g, eps, out, r, h, pr);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- RMSNorm bwd
// yhat = y r; dg += dz * yhat; dy = r (g dz - yhat mean_j(g dz yhat))
template <typename TY>
__global__ void rmsnorm_bwd_kernel(const float* __restrict__ dz, const TY* __restrict__ y,
                                   const float* __restrict__ r, const float* __restrict__ g,
                                   __nv_bfloat16* dy, const __nv_bfloat16* add,
                                   float* __restrict__ dg_part, long long n, int h, int rpb,
                                   int nslots, long long slot_stride) {
  __shared__ float red[33];
  const int nchunk = h / 8;
  float gv[NORM_CHUNKS][8], acc[NORM_CHUNKS][8];
#pragma unroll
  for (int i = 0; i < NORM_CHUNKS; ++i) {
    const int c = threadIdx.x + i * blockDim.x;
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[i][k] = 0.f;
    if (c < nchunk) load8(g + c * 8, gv[i]);
  }
  const long long r0 = (long long)blockIdx.x * rpb;
  const long long r1 = min(n, r0 + rpb);
  // Row `row`'s dz (summed over the slots, in slot order) and y into registers.
  auto load_row = [&](long long row, float (&d)[NORM_CHUNKS][8], float (&yv)[NORM_CHUNKS][8]) {
#pragma unroll
    for (int i = 0; i < NORM_CHUNKS; ++i) {
      const int c = threadIdx.x + i * blockDim.x;
      if (c < nchunk) {
        load8(dz + row * h + c * 8, d[i]);
        for (int q = 1; q < nslots; ++q) {  // owner-side sum of the fused reduce-scatter
          float e[8];
          load8(dz + q * slot_stride + row * h + c * 8, e);
#pragma unroll
          for (int k = 0; k < 8; ++k) d[i][k] += e[k];
        }
        load8(y + row * h + c * 8, yv[i]);
      }
    }
  };
  float dn[NORM_CHUNKS][8], yn[NORM_CHUNKS][8];  // the next row, loaded one row ahead
  if (r0 < r1) load_row(r0, dn, yn);
  for (long long row = r0; row < r1; ++row) {
    const float rr = r[row];
    float d[NORM_CHUNKS][8], yh[NORM_CHUNKS][8];
#pragma unroll
    for (int i = 0; i < NORM_CHUNKS; ++i)
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        d[i][k] = dn[i][k];
        yh[i][k] = yn[i][k];
      }
    if (row + 1 < r1) load_row(row + 1, dn, yn);  // in flight across this row's reduction
    float dot = 0.f;
#pragma unroll
    for (int i = 0; i < NORM_CHUNKS; ++i) {
      const int c = threadIdx.x + i * blockDim.x;
      if (c < nchunk) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          yh[i][k] *= rr;
          dot += gv[i][k] * d[i][k] * yh[i][k];
          acc[i][k] += d[i][k] * yh[i][k];
        }
      }
    }
    if (dy != nullptr) {
      const float mean = block_sum(dot, red) / (float)h;
#pragma unroll
      for (int i = 0; i < NORM_CHUNKS; ++i) {
        const int c = threadIdx.x + i * blockDim.x;
        if (c < nchunk) {
          float o[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) o[k] = rr * (gv[i][k] * d[i][k] - yh[i][k] * mean);
          if (add != nullptr) {  // residual branch (may alias dy: same thread, read first)
            float a8[8];
            load8(add + row * h + c * 8, a8);
#pragma unroll
            for (int k = 0; k < 8; ++k) o[k] += a8[k];
          }
          store8(dy + row * h + c * 8, o);
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < NORM_CHUNKS; ++i) {
    const int c = threadIdx.x + i * blockDim.x;
    if (c < nchunk) {
      float* p = dg_part + (long long)blockIdx.x * h + c * 8;
      *reinterpret_cast<float4*>(p) = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
      *reinterpret_cast<float4*>(p + 4) = make_float4(acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
    }
  }
}

cudaError_t launch_rmsnorm_bwd(const float* dz, const void* y, bool y_f32, const float* r,
                               const float* g, __nv_bfloat16* dy, float* dg_part, long long n,
                               int h, int rpb, cudaStream_t s, const __nv_bfloat16* add,
                               int nslots, long long slot_stride) {
  const unsigned nb = (unsigned)((n + rpb - 1) / rpb);
  if (nb == 0) return cudaSuccess;
  const int t = norm_threads(h);
  if (y_f32)
    rmsnorm_bwd_kernel<float>
        <<<nb, t, 0, s>>>(dz, (const float*)y, r, g, dy, add, dg_part, n, h, rpb, nslots,
                          slot_stride);
  else
    rmsnorm_bwd_kernel<__nv_bfloat16>
        <<<nb, t, 0, s>>>(dz, (const __nv_bfloat16*)y, r, g, dy, add, dg_part, n, h, rpb,
                          nslots, slot_stride);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- RoPE table
// (cos, sin) of the Llama rotate-half angle pos * theta^(-2i/128) for
// pos < T, i < 64, evaluated in fp64 and rounded once to fp32 (read by the
// q/k projection epilogues instead of an fp32 powf + sincosf per element).
__global__ void rope_table_kernel(float2* __restrict__ tab, int T, double theta) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= T * 64) return;
  const int pos = idx >> 6, i = idx & 63;
  const double ang = (double)pos * pow(theta, -2.0 * (double)i / 128.0);
  double sn, cs;
  sincos(ang, &sn, &cs);
  tab[idx] = make_float2((float)cs, (float)sn);
}

cudaError_t launch_rope_table(float2* tab, int T, float theta, cudaStream_t s) {
  if (T <= 0) return cudaSuccess;
  rope_table_kernel<<<(T * 64 + 255) / 256, 256, 0, s>>>(tab, T, (double)theta);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- peer barrier
// Rank `rank` publishes `epoch` into slot `rank` of every rank's signal array
// (release at system scope: this stream's earlier kernels, including their
// NVLink stores into peer buffers, are complete and visible first), then waits
// until its own array holds >= epoch in all `world` slots (acquire).  Thread q
// handles peer q.  A peer missing for ~20 s sets EE_ERR_PEER instead of hanging.
__global__ void peer_barrier_kernel(PeerSig sig, int rank, int world, unsigned epoch,
                                    DevStatus* st) {
  const int q = threadIdx.x;
  if (q >= world) return;
  __threadfence_system();
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(sig.p[q] + rank), "r"(epoch) : "memory");
  const int* mine = sig.p[rank] + q;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (true) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(mine) : "memory");
    if ((int)(v - epoch) >= 0) break;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 20000000000ull) {
      set_status(st, 12 /* EE_ERR_PEER */, q);
      break;
    }
    __nanosleep(256);
  }
}

cudaError_t launch_peer_barrier(int* const* sig, int rank, int world, unsigned epoch,
                                DevStatus* st, cudaStream_t s) {
  PeerSig ps{};
  for (int q = 0; q < world && q < MAX_PEERS; ++q) ps.p[q] = sig[q];
  peer_barrier_kernel<<<1, 32, 0, s>>>(ps, rank, world, epoch, st);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- gain grad
// dg_a = sum_t du_t * (x_t r_t)   (no dx: the backbone is frozen)
__global__ void gain_grad_kernel(const float* __restrict__ du, const __nv_bfloat16* __restrict__ x,
                                 const float* __restrict__ r, float* __restrict__ dg_part,
                                 long long n, int h, int rpb) {
  const int nchunk = h / 8;
  float acc[NORM_CHUNKS][8];
#pragma unroll
  for (int i = 0; i < NORM_CHUNKS; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[i][k] = 0.f;
  const long long r0 = (long long)blockIdx.x * rpb;
  const long long r1 = min(n, r0 + rpb);
  for (long long row = r0; row < r1; ++row) {
    const float rr = r[row];
#pragma unroll
    for (int i = 0; i < NORM_CHUNKS; ++i) {
      const int c = threadIdx.x + i * blockDim.x;
      if (c < nchunk) {
        float d[8], xv[8];
        load8(du + row * h + c * 8, d);
        load8(x + row * h + c * 8, xv);
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[i][k] += d[k] * (xv[k] * rr);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < NORM_CHUNKS; ++i) {
    const int c = threadIdx.x + i * blockDim.x;
    if (c < nchunk) {
      float* p = dg_part + (long long)blockIdx.x * h + c * 8;
      *reinterpret_cast<float4*>(p) = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
      *reinterpret_cast<float4*>(p + 4) = make_float4(acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
    }
  }
}

cudaError_t launch_gain_grad(const float* du, const __nv_bfloat16* x, const float* r,
                             float* dg_part, long long n, int h, int rpb, cudaStream_t s) {
  const unsigned nb = (unsigned)((n + rpb - 1) / rpb);
  if (nb == 0) return cudaSuccess;
  gain_grad_kernel<<<nb, norm_threads(h), 0, s>>>(du, x, r, dg_part, n, h, rpb);
  return cudaGetLastError();
}

// Column sums of [nparts x h] partials in part order (deterministic).
__global__ void reduce_cols_kernel(const float* __restrict__ part, int nparts, int h,
                                   float* __restrict__ out, int accumulate) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= h) return;
  float s = 0.f;
  for (int p = 0; p < nparts; ++p) s += part[(long long)p * h + c];
  out[c] = accumulate ? out[c] + s : s;
}

cudaError_t launch_reduce_cols(const float* part, int nparts, int h, float* out, int accumulate,
                               cudaStream_t s) {
  reduce_cols_kernel<<<(h + 255) / 256, 256, 0, s>>>(part, nparts, h, out, accumulate);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- CE finalize
// Merge the per-V-tile (max, sum-exp, argmax) partials of each row:
//   m = max_j m_j; s = sum_j s_j exp(m_j - m); lse = m + ln s;
//   loss_t = lse - S[y_t]; conf_t = 1/s (max softmax prob);
//   argmax = the argmax of the first tile attaining m (lowest index, A9);
//   coef_t = alpha_i w_t / W (the dS scale).
__global__ void ce_finalize_kernel(const float* __restrict__ pm, const float* __restrict__ ps,
                                   const int32_t* __restrict__ pi, const float* __restrict__ tl,
                                   const int32_t* __restrict__ targets, int nb, long long n,
                                   const long long* __restrict__ valid_count, float alpha,
                                   float* __restrict__ lse, float* __restrict__ coef,
                                   float* aux_lse, float* aux_loss, int32_t* aux_argmax,
                                   float* aux_conf, float* __restrict__ loss_part,
                                   float* __restrict__ wsum_part) {
  __shared__ double red[33];
  const long long row = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  double lossv = 0.0, wsum = 0.0;
  if (row < n) {
    float m = -INFINITY;
    for (int j = 0; j < nb; ++j) m = fmaxf(m, pm[(long long)j * n + row]);
    float s = 0.f;
    int am = INT_MAX;
    for (int j = 0; j < nb; ++j) {
      const float mj = pm[(long long)j * n + row];
      s += ps[(long long)j * n + row] * expf(mj - m);
      if (mj == m && am == INT_MAX) am = pi[(long long)j * n + row];
    }
    const float l = m + logf(s);
    const int y = targets[row];
    const bool valid = y >= 0;
    const float lt = valid ? l - tl[row] : 0.f;  // tl never read for ignored rows
    lse[row] = l;
    if (aux_lse) aux_lse[row] = l;
    if (aux_loss) aux_loss[row] = lt;
    if (aux_argmax) aux_argmax[row] = am;
    if (aux_conf) aux_conf[row] = 1.0f / s;
    if (wsum_part) {  // confidence weights w_t = c_t = 1/s, detached
      const float w = valid ? 1.0f / s : 0.f;
      coef[row] = w;  // scaled by alpha / sum(w) in ce_coef_scale
      lossv = (double)w * (double)lt;
      wsum = (double)w;
    } else {
      const long long W = *valid_count;
      coef[row] = (valid && W > 0) ? alpha / (float)W : 0.f;
      lossv = (double)lt;
    }
  }
  lossv = block_sum(lossv, red);
  if (threadIdx.x == 0) loss_part[blockIdx.x] = (float)lossv;
  if (wsum_part) {
    wsum = block_sum(wsum, red);
    if (threadIdx.x == 0) wsum_part[blockIdx.x] = (float)wsum;
  }
}

cudaError_t launch_ce_finalize(const float* pm, const float* ps, const int32_t* pi,
                               const float* tl, const int32_t* targets, int nb, long long n,
                               const long long* valid_count, float alpha, float* lse, float* coef,
                               float* aux_lse, float* aux_loss, int32_t* aux_argmax,
                               float* aux_conf, float* loss_part, float* wsum_part, int nblocks,
                               cudaStream_t s) {
  if (nblocks == 0) return cudaSuccess;
  ce_finalize_kernel<<<nblocks, FINALIZE_THREADS, 0, s>>>(pm, ps, pi, tl, targets, nb, n,
                                                          valid_count, alpha, lse, coef, aux_lse,
                                                          aux_loss, aux_argmax, aux_conf,
                                                          loss_part, wsum_part);
  return cudaGetLastError();
}

// a7 without a second GEMM: the a5 epilogue stored P~[t][v] = exp(S_tv - m_tj)
// (fp16, m_tj = row t's max over its 256-column tile j, kept in pm[j][t]);
// here, in place, dS_tv = coef_t (P~_tv exp(m_tj - lse_t) - 1[v = y_t]) as
// bf16 (the softmax-CE gradient; coef_t = alpha w_t / W).  The target
// column is recomputed from the fp32 target logit, exp(S_ty - lse_t) - 1, so
// confident rows (p_y -> 1) keep full relative precision.  One CTA per row,
// 16-byte accesses.
__global__ void ce_ds_from_p_kernel(__nv_bfloat16* __restrict__ ds, int Vl, long long n,
                                    const float* __restrict__ pm, const float* __restrict__ lse,
                                    const float* __restrict__ coef,
                                    const int32_t* __restrict__ targets, int vocab_begin,
                                    const float* __restrict__ tgt_logit) {
  const long long row = blockIdx.x;
  const float l = lse[row], cf = coef[row];
  const int y = targets[row] - vocab_begin;
  __nv_bfloat16* drow = ds + row * (long long)Vl;
  const int nch = Vl / 8;
  constexpr int U = 4;  // chunks per thread per iteration: their loads are issued together
  for (int c0 = threadIdx.x; c0 < nch; c0 += U * blockDim.x) {
    uint4 q[U];
    float f[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c = c0 + u * blockDim.x;
      if (c < nch) {
        q[u] = *reinterpret_cast<const uint4*>(drow + c * 8);
        f[u] = pm[(long long)(c >> 5) * n + row];  // 256-column tile of these 8 columns
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c = c0 + u * blockDim.x;
      if (c >= nch) continue;
      const float fu = cf * __expf(f[u] - l);
      const uint32_t w[4] = {q[u].x, q[u].y, q[u].z, q[u].w};
      float d[8];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 p2 = __half22float2(*reinterpret_cast<const __half2*>(&w[k]));
        d[2 * k] = fu * p2.x;
        d[2 * k + 1] = fu * p2.y;
      }
      const int yo = y - c * 8;
      if (yo >= 0 && yo < 8) d[yo] = cf * (__expf(tgt_logit[row] - l) - 1.0f);
      uint4 o;
      o.x = pack_bf16(d[0], d[1]);
      o.y = pack_bf16(d[2], d[3]);
      o.z = pack_bf16(d[4], d[5]);
      o.w = pack_bf16(d[6], d[7]);
      *reinterpret_cast<uint4*>(drow + c * 8) = o;
    }
  }
}

cudaError_t launch_ce_ds_from_p(__nv_bfloat16* ds, int Vl, long long n, const float* pm,
                                const float* lse, const float* coef, const int32_t* targets,
                                int vocab_begin, const float* tgt_logit, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  ce_ds_from_p_kernel<<<(unsigned)n, 256, 0, s>>>(ds, Vl, n, pm, lse, coef, targets, vocab_begin,
                                                 tgt_logit);
  return cudaGetLastError();
}

// L_i = sum_t w_t loss_t / W (A4, A16); non-finite -> EE_ERR_DIVERGED.
__global__ void loss_reduce_kernel(const float* __restrict__ part, int nparts,
                                   const long long* __restrict__ valid_count,
                                   const float* __restrict__ wsum_part, float* wsum_out,
                                   float* loss_out, DevStatus* st, int exit_index, int normalize) {
  __shared__ double red[33];
  double s = 0.0, ws = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) {
    s += (double)part[i];
    if (wsum_part) ws += (double)wsum_part[i];
  }
  s = block_sum(s, red);
  if (wsum_part) ws = block_sum(ws, red);
  if (threadIdx.x == 0) {
    const double W = wsum_part ? ws : (double)*valid_count;
    const float L = !normalize ? (float)s : (W > 0 ? (float)(s / W) : 0.f);
    *loss_out = L;
    if (wsum_out) *wsum_out = (float)W;
    if (!isfinite(L)) set_status(st, 7 /*EE_ERR_DIVERGED*/, exit_index);
  }
}

cudaError_t launch_loss_reduce(const float* loss_part, int nparts, const long long* valid_count,
                               const float* wsum_part, float* wsum_out, float* loss_out,
                               DevStatus* st, int exit_index, cudaStream_t s, bool normalize) {
  loss_reduce_kernel<<<1, 1024, 0, s>>>(loss_part, nparts, valid_count, wsum_part, wsum_out,
                                        loss_out, st, exit_index, normalize ? 1 : 0);
  return cudaGetLastError();
}

// coef_t = alpha * w_t / sum_t w_t  (confidence weighting; w_t stored in coef);
// wsum == NULL: alpha * w_t (the normaliser is applied later, ee_normalize_exit)
__global__ void ce_coef_scale_kernel(float* coef, long long n, float alpha, const float* wsum) {
  const long long row = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= n) return;
  if (wsum == nullptr) {
    coef[row] = alpha * coef[row];
    return;
  }
  const float W = *wsum;
  coef[row] = W > 0.f ? alpha * coef[row] / W : 0.f;
}

cudaError_t launch_ce_coef_scale(float* coef, long long n, float alpha, const float* wsum,
                                 cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  ce_coef_scale_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(coef, n, alpha, wsum);
  return cudaGetLastError();
}

// x[i] *= 1 / *den  (den a device scalar; 0 -> x = 0)
__global__ void scale_by_inv_kernel(float* __restrict__ x, long long n, const float* __restrict__ den) {
  const float d = *den;
  const float f = d > 0.f ? 1.0f / d : 0.f;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    x[i] *= f;
}

cudaError_t launch_scale_by_inv(float* x, long long n, const float* den, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const unsigned nb = (unsigned)std::min<long long>((n + 255) / 256, 148LL * 16);
  scale_by_inv_kernel<<<nb, 256, 0, s>>>(x, n, den);
  return cudaGetLastError();
}


// ---------------------------------------------------------------- vocab parallel CE
// Rank r holds W_out rows [vb, ve).  Per row it merges its own V tiles into
// (m_r, s_r = sum exp(S - m_r), argmax_r, S[y] if y in [vb, ve) else 0); the
// caller all-reduces MAX over the (m, argmax) key and then SUM over
// (s_r exp(m_r - m), S[y]) -- the distributed softmax-CE of north_star.
__device__ __forceinline__ long long vp_make_key(float m, int idx) {
  uint32_t u = __float_as_uint(m);
  u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  const unsigned long long k =
      ((unsigned long long)u << 32) | (unsigned long long)(0xFFFFFFFFu - (uint32_t)idx);
  return (long long)(k ^ 0x8000000000000000ull);
}
__device__ __forceinline__ void vp_split_key(long long key, float& m, int& idx) {
  const unsigned long long k = (unsigned long long)key ^ 0x8000000000000000ull;
  uint32_t u = (uint32_t)(k >> 32);
  u = (u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u;
  m = __uint_as_float(u);
  idx = (int)(0xFFFFFFFFu - (uint32_t)(k & 0xFFFFFFFFull));
}

__global__ void vp_local_merge_kernel(const float* __restrict__ pm, const float* __restrict__ ps,
                                      const int32_t* __restrict__ pi, const float* __restrict__ tl,
                                      const int32_t* __restrict__ targets, int nb, long long n,
                                      int vb, int ve, long long* key, float* m_loc, float* sums) {
  const long long row = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= n) return;
  float m = -INFINITY;
  for (int j = 0; j < nb; ++j) m = fmaxf(m, pm[(long long)j * n + row]);
  float s = 0.f;
  int am = INT_MAX;
  for (int j = 0; j < nb; ++j) {
    const float mj = pm[(long long)j * n + row];
    s += ps[(long long)j * n + row] * expf(mj - m);
    if (mj == m && am == INT_MAX) am = pi[(long long)j * n + row];
  }
  const int y = targets[row];
  key[row] = vp_make_key(m, am);
  m_loc[row] = m;
  sums[2 * row] = s;
  sums[2 * row + 1] = (y >= vb && y < ve) ? tl[row] : 0.f;
}

cudaError_t launch_vp_local_merge(const float* pm, const float* ps, const int32_t* pi,
                                  const float* tl, const int32_t* targets, int nb, long long n,
                                  int vocab_begin, int vocab_end, long long* key, float* m_loc,
                                  float* sums, cudaStream_t s) {
  vp_local_merge_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(
      pm, ps, pi, tl, targets, nb, n, vocab_begin, vocab_end, key, m_loc, sums);
  return cudaGetLastError();
}

__global__ void vp_rescale_kernel(const long long* __restrict__ key, const float* __restrict__ m_loc,
                                  float* sums, long long n) {
  const long long row = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= n) return;
  float m;
  int idx;
  vp_split_key(key[row], m, idx);
  sums[2 * row] *= expf(m_loc[row] - m);
}

cudaError_t launch_vp_rescale(const long long* key_global, const float* m_loc, float* sums,
                              long long n, cudaStream_t s) {
  vp_rescale_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(key_global, m_loc, sums, n);
  return cudaGetLastError();
}

__global__ void vp_finalize_kernel(const long long* __restrict__ key, const float* __restrict__ sums,
                                   const int32_t* __restrict__ targets, long long n,
                                   const long long* __restrict__ valid_count, float alpha,
                                   float* __restrict__ lse, float* __restrict__ coef,
                                   float* aux_lse, float* aux_loss, int32_t* aux_argmax,
                                   float* aux_conf, float* __restrict__ loss_part,
                                   float* __restrict__ wsum_part) {
  __shared__ double red[33];
  const long long row = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  double lossv = 0.0, wsum = 0.0;
  if (row < n) {
    float m;
    int am;
    vp_split_key(key[row], m, am);
    const float s = sums[2 * row];
    const float l = m + logf(s);
    const int y = targets[row];
    const bool valid = y >= 0;
    const float lt = valid ? l - sums[2 * row + 1] : 0.f;
    lse[row] = l;
    if (aux_lse) aux_lse[row] = l;
    if (aux_loss) aux_loss[row] = lt;
    if (aux_argmax) aux_argmax[row] = am;
    if (aux_conf) aux_conf[row] = 1.0f / s;
    if (wsum_part) {
      const float w = valid ? 1.0f / s : 0.f;
      coef[row] = w;
      lossv = (double)w * (double)lt;
      wsum = (double)w;
    } else {
      const long long W = *valid_count;
      coef[row] = (valid && W > 0) ? alpha / (float)W : 0.f;
      lossv = (double)lt;
    }
  }
  lossv = block_sum(lossv, red);
  if (threadIdx.x == 0) loss_part[blockIdx.x] = (float)lossv;
  if (wsum_part) {
    wsum = block_sum(wsum, red);
    if (threadIdx.x == 0) wsum_part[blockIdx.x] = (float)wsum;
  }
}

cudaError_t launch_vp_finalize(const long long* key_global, const float* sums,
                               const int32_t* targets, long long n, const long long* valid_count,
                               float alpha, float* lse, float* coef, float* aux_lse,
                               float* aux_loss, int32_t* aux_argmax, float* aux_conf,
                               float* loss_part, float* wsum_part, int nblocks, cudaStream_t s) {
  if (nblocks == 0) return cudaSuccess;
  vp_finalize_kernel<<<nblocks, FINALIZE_THREADS, 0, s>>>(key_global, sums, targets, n,
                                                          valid_count, alpha, lse, coef, aux_lse,
                                                          aux_loss, aux_argmax, aux_conf,
                                                          loss_part, wsum_part);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- early exit (inference)
// first_exit[t] = lowest exit index i with conf_i[t] >= tau, else -1 (
// tau = 1 disables early exits).
struct ConfPtrs {
  const float* p[64];
};
__global__ void first_exit_kernel(ConfPtrs c, int E, long long n, float tau, int32_t* out) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  griddep_wait();  // PDL launch (launch_first_exit)
  if (t >= n) return;
  int f = -1;
  for (int i = 0; i < E; ++i)
    if (c.p[i][t] >= tau) {
      f = i;
      break;
    }
  out[t] = f;
}

cudaError_t launch_first_exit(const float* const* conf, int E, long long n, float tau,
                              int32_t* out, cudaStream_t s) {
  ConfPtrs c;
  for (int i = 0; i < E && i < 64; ++i) c.p[i] = conf[i];
  return launch_pdl(first_exit_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, s, c, E,
                    n, tau, out);
}

// ---------------------------------------------------------------- transpose
// dst[C x R] = src[R x C]^T (bf16), 64 x 64 tiles through shared memory:
// 128-byte coalesced reads and writes.  Gives the weight-gradient GEMMs a
// K-major copy of their token-major activation operand (u, z, dy), so their
// A operand takes the K-major UMMA path.
// dst[c][r] = src[r][c] (rscale == NULL) or bf16(src[r][c] * rscale[r]) -- the
// latter is x^ = x r (RMSNorm before its gain), transposed, for the gain identity
__global__ void transpose_bf16_kernel(const __nv_bfloat16* __restrict__ src,
                                      __nv_bfloat16* __restrict__ dst, long long R, int C,
                                      long long ldd, const float* __restrict__ rscale) {
  // 64 x 64 tile; 16-byte global loads and stores (8 bf16 per access), rows of
  // the smem tile padded to 33 words so the column gathers are 2-way conflicted
  __shared__ uint32_t tile[64][33];
  const long long r0 = (long long)blockIdx.y * 64;
  const int c0 = blockIdx.x * 64;
  const bool fast = (C % 8) == 0;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int ch = threadIdx.x + h * 256;  // 512 chunks of 8 columns
    const int i = ch >> 3, j = (ch & 7) * 8;
    const long long r = r0 + i;
    const int c = c0 + j;
    uint32_t w[4] = {0u, 0u, 0u, 0u};
    if (r < R) {
      if (fast && c + 8 <= C) {
        const uint4 q = *reinterpret_cast<const uint4*>(src + r * C + c);
        w[0] = q.x; w[1] = q.y; w[2] = q.z; w[3] = q.w;
      } else {
        __nv_bfloat16 e[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) e[k] = (c + k < C) ? src[r * C + c + k] : __float2bfloat16_rn(0.f);
#pragma unroll
        for (int k = 0; k < 4; ++k) w[k] = *reinterpret_cast<const uint32_t*>(&e[2 * k]);
      }
      if (rscale != nullptr) {
        const float rr = rscale[r];
#pragma unroll
        for (int k = 0; k < 4; ++k)
          w[k] = pack_bf16(__uint_as_float(w[k] << 16) * rr, __uint_as_float(w[k] & 0xFFFF0000u) * rr);
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) tile[i][j / 2 + k] = w[k];
  }
  __syncthreads();
  const __nv_bfloat16* tb = reinterpret_cast<const __nv_bfloat16*>(&tile[0][0]);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int ch = threadIdx.x + h * 256;
    const int oc = ch >> 3, rr = (ch & 7) * 8;  // output row c0 + oc, rows rr..rr+7 of the tile
    const int c = c0 + oc;
    if (c >= C) continue;
    const long long r = r0 + rr;
    if (r >= R) continue;
    __nv_bfloat16 e[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) e[k] = tb[(rr + k) * 66 + oc];
    __nv_bfloat16* d = dst + (long long)c * ldd + r;
    if (r + 8 <= R && ((reinterpret_cast<uintptr_t>(d) & 15) == 0)) {
      uint4 q;
      q.x = *reinterpret_cast<const uint32_t*>(&e[0]);
      q.y = *reinterpret_cast<const uint32_t*>(&e[2]);
      q.z = *reinterpret_cast<const uint32_t*>(&e[4]);
      q.w = *reinterpret_cast<const uint32_t*>(&e[6]);
      *reinterpret_cast<uint4*>(d) = q;
    } else {
      for (int k = 0; k < 8 && r + k < R; ++k) d[k] = e[k];
    }
  }
}

cudaError_t launch_transpose_bf16(const __nv_bfloat16* src, __nv_bfloat16* dst, long long R, int C,
                                  long long ldd, cudaStream_t s, const float* rscale) {
  if (R == 0 || C == 0) return cudaSuccess;
  dim3 grid((C + 63) / 64, (unsigned)((R + 63) / 64));
  transpose_bf16_kernel<<<grid, 256, 0, s>>>(src, dst, R, C, ldd, rscale);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- optimizer
static inline unsigned ew_blocks(long long n4) {
  long long b = (n4 + 255) / 256;
  const long long cap = (long long)num_sms() * 16;
  return (unsigned)(b < cap ? (b > 0 ? b : 1) : cap);
}

// Adam (A14), 4 elements per thread-iteration.
__global__ void adam_kernel(float* __restrict__ th, __nv_bfloat16* op_bf16, float* op_f32,
                            const float* __restrict__ gr, float* __restrict__ m,
                            float* __restrict__ v, long long n4, float lr, float b1, float b2,
                            float eps, float wd, float bc1, float bc2, float gs) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x) {
    float4 t = reinterpret_cast<float4*>(th)[i];
    const float4 g4 = reinterpret_cast<const float4*>(gr)[i];
    float4 m4 = reinterpret_cast<float4*>(m)[i];
    float4 v4 = reinterpret_cast<float4*>(v)[i];
    float* tp = &t.x;
    const float* gp = &g4.x;
    float* mp = &m4.x;
    float* vp = &v4.x;
    const AdamScal sc{lr, b1, b2, eps, wd, bc1, bc2, gs};
#pragma unroll
    for (int k = 0; k < 4; ++k) adam_update(tp[k], mp[k], vp[k], gp[k], sc);
    reinterpret_cast<float4*>(th)[i] = t;
    reinterpret_cast<float4*>(m)[i] = m4;
    reinterpret_cast<float4*>(v)[i] = v4;
    if (op_bf16) {
      uint2 q;
      q.x = pack_bf16(t.x, t.y);
      q.y = pack_bf16(t.z, t.w);
      reinterpret_cast<uint2*>(op_bf16)[i] = q;
    }
    if (op_f32) reinterpret_cast<float4*>(op_f32)[i] = t;
  }
}

// Sharded Adam of the fused data-parallel path (ZeRO-1; include/ee.h
// ee_adam_update_sharded): this rank owns n4*4 elements of one tensor.  Its
// gradient is the rank-ordered sum of the P slots [P][n] that every rank's
// backward stored here (the reduce-scatter's owner-side sum), the update is
// adam_kernel's arithmetic, and the new operand values (bf16 matrices / fp32
// gains) are stored into every rank's operand tensor at element offset off4*4
// (the all-gather, as NVLink stores).
__global__ void adam_sharded_kernel(float* __restrict__ th, const float* __restrict__ slots,
                                    int P, float* __restrict__ m, float* __restrict__ v,
                                    long long n4, OpPeers op, long long off4, float lr, float b1,
                                    float b2, float eps, float wd, float bc1, float bc2,
                                    float gs, const float* __restrict__ div) {
  // dynamic token weights under DP: divide by the global sum of weights
  // (ee_normalize_exit's arithmetic: x *= 1/d, 0 if d <= 0)
  float fdiv = 1.f;
  if (div) {
    const float d = *div;
    fdiv = d > 0.f ? 1.0f / d : 0.f;
  }
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x) {
    float4 t = reinterpret_cast<float4*>(th)[i];
    float4 g4 = reinterpret_cast<const float4*>(slots)[i];
    for (int r = 1; r < P; ++r) {
      const float4 e = reinterpret_cast<const float4*>(slots)[(long long)r * n4 + i];
      g4.x += e.x; g4.y += e.y; g4.z += e.z; g4.w += e.w;
    }
    if (div) {
      g4.x *= fdiv; g4.y *= fdiv; g4.z *= fdiv; g4.w *= fdiv;
    }
    float4 m4 = reinterpret_cast<float4*>(m)[i];
    float4 v4 = reinterpret_cast<float4*>(v)[i];
    float* tp = &t.x;
    const float* gp = &g4.x;
    float* mp = &m4.x;
    float* vp = &v4.x;
    const AdamScal sc{lr, b1, b2, eps, wd, bc1, bc2, gs};
#pragma unroll
    for (int k = 0; k < 4; ++k) adam_update(tp[k], mp[k], vp[k], gp[k], sc);
    reinterpret_cast<float4*>(th)[i] = t;
    reinterpret_cast<float4*>(m)[i] = m4;
    reinterpret_cast<float4*>(v)[i] = v4;
    if (op.f32) {
#pragma unroll
      for (int q = 0; q < MAX_PEERS; ++q)
        if (q < op.n) reinterpret_cast<float4*>(op.p[q])[off4 + i] = t;
    } else {
      uint2 w;
      w.x = pack_bf16(t.x, t.y);
      w.y = pack_bf16(t.z, t.w);
#pragma unroll
      for (int q = 0; q < MAX_PEERS; ++q)
        if (q < op.n) reinterpret_cast<uint2*>(op.p[q])[off4 + i] = w;
    }
  }
}

cudaError_t launch_adam_sharded(float* theta, const float* slots, int P, float* m, float* v,
                                long long n, const OpPeers& op, long long off, float lr, float b1,
                                float b2, float eps, float wd, float bc1, float bc2, float gs,
                                cudaStream_t s, const float* div) {
  if (n == 0) return cudaSuccess;
  const long long n4 = n / 4;
  adam_sharded_kernel<<<ew_blocks(n4), 256, 0, s>>>(theta, slots, P, m, v, n4, op, off / 4, lr,
                                                    b1, b2, eps, wd, bc1, bc2, gs, div);
  return cudaGetLastError();
}

cudaError_t launch_adam(float* theta, __nv_bfloat16* op_bf16, float* op_f32, const float* grad,
                        float* m, float* v, long long n, float lr, float b1, float b2, float eps,
                        float wd, float bc1, float bc2, float gscale, cudaStream_t s) {
  const long long n4 = n / 4;
  adam_kernel<<<ew_blocks(n4), 256, 0, s>>>(theta, op_bf16, op_f32, grad, m, v, n4, lr, b1, b2,
                                            eps, wd, bc1, bc2, gscale);
  return cudaGetLastError();
}

__global__ void sgd_kernel(float* __restrict__ th, __nv_bfloat16* op_bf16, float* op_f32,
                           const float* __restrict__ gr, float* buf, long long n4, float lr,
                           float mom, float gs) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x) {
    float4 t = reinterpret_cast<float4*>(th)[i];
    float4 g4 = reinterpret_cast<const float4*>(gr)[i];
    float* tp = &t.x;
    float* gp = &g4.x;
    if (buf) {
      float4 b4 = reinterpret_cast<float4*>(buf)[i];
      float* bp = &b4.x;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        bp[k] = mom * bp[k] + gs * gp[k];
        gp[k] = bp[k];
      }
      reinterpret_cast<float4*>(buf)[i] = b4;
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) gp[k] *= gs;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) tp[k] -= lr * gp[k];
    reinterpret_cast<float4*>(th)[i] = t;
    if (op_bf16) {
      uint2 q;
      q.x = pack_bf16(t.x, t.y);
      q.y = pack_bf16(t.z, t.w);
      reinterpret_cast<uint2*>(op_bf16)[i] = q;
    }
    if (op_f32) reinterpret_cast<float4*>(op_f32)[i] = t;
  }
}

cudaError_t launch_sgd(float* theta, __nv_bfloat16* op_bf16, float* op_f32, const float* grad,
                       float* buf, long long n, float lr, float mom, float gscale, cudaStream_t s) {
  const long long n4 = n / 4;
  sgd_kernel<<<ew_blocks(n4), 256, 0, s>>>(theta, op_bf16, op_f32, grad, buf, n4, lr, mom, gscale);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- initialisers
// Copy: deep copy of the source module, widened to the fp32 master
// and narrowed to the bf16 operand (exact when the source is bf16).
template <typename TS>
__global__ void copy_cast_kernel(const TS* __restrict__ src, float* master, __nv_bfloat16* op_bf16,
                                 float* op_f32, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const float v = (float)src[i];
    if (master) master[i] = v;
    if (op_bf16) op_bf16[i] = __float2bfloat16_rn(v);
    if (op_f32) op_f32[i] = v;
  }
}

cudaError_t launch_copy_cast(const void* src, bool src_f32, float* master, __nv_bfloat16* op_bf16,
                             float* op_f32, long long n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  if (src_f32)
    copy_cast_kernel<float><<<ew_blocks(n / 4 + 1), 256, 0, s>>>((const float*)src, master,
                                                                  op_bf16, op_f32, n);
  else
    copy_cast_kernel<__nv_bfloat16><<<ew_blocks(n / 4 + 1), 256, 0, s>>>(
        (const __nv_bfloat16*)src, master, op_bf16, op_f32, n);
  return cudaGetLastError();
}

// Philox4x32-10 (Salmon et al. 2011), counter = (i, 0, stream lo, stream hi),
// key = seed; Box-Muller on the 4 outputs -> 4 N(0,1) samples.
__device__ __forceinline__ void philox4x32_10(uint32_t (&c)[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c[0]), lo0 = 0xD2511F53u * c[0];
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]), lo1 = 0xCD9E8D57u * c[2];
    const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

__global__ void random_normal_kernel(uint64_t seed, uint64_t sid, float std, float* master,
                                     __nv_bfloat16* op_bf16, long long n) {
  const long long n4 = (n + 3) / 4;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x) {
    uint32_t c[4] = {(uint32_t)i, (uint32_t)(i >> 32), (uint32_t)sid, (uint32_t)(sid >> 32)};
    philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
    float z[4];
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      const float u1 = ((float)c[2 * p] + 1.0f) * 2.3283064365386963e-10f;  // (0, 1]
      const float u2 = (float)c[2 * p + 1] * 2.3283064365386963e-10f;       // [0, 1)
      const float rad = sqrtf(-2.0f * logf(u1));
      float sn, cs;
      sincospif(2.0f * u2, &sn, &cs);
      z[2 * p] = rad * cs;
      z[2 * p + 1] = rad * sn;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const long long j = i * 4 + k;
      if (j < n) {
        const float w = std * z[k];
        const __nv_bfloat16 b = __float2bfloat16_rn(w);
        // master on the bf16 grid so operand == master exactly at t = 0
        if (master) master[j] = __bfloat162float(b);
        if (op_bf16) op_bf16[j] = b;
      }
    }
  }
}

cudaError_t launch_random_normal(uint64_t seed, uint64_t stream_id, float std, float* master,
                                 __nv_bfloat16* op_bf16, long long n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  random_normal_kernel<<<ew_blocks(n / 4 + 1), 256, 0, s>>>(seed, stream_id, std, master, op_bf16,
                                                            n);
  return cudaGetLastError();
}

__global__ void fill_kernel(float* a, float* b, long long n, float v) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    if (a) a[i] = v;
    if (b) b[i] = v;
  }
}

cudaError_t launch_fill(float* master, float* op_f32, long long n, float value, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  fill_kernel<<<ew_blocks(n / 4 + 1), 256, 0, s>>>(master, op_f32, n, value);
  return cudaGetLastError();
}

}  // namespace ee
