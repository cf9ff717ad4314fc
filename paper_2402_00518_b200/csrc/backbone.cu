// backbone.cu -- the frozen backbone's partial forward (NEXT #3; P:258-260,
// PAPER.md §2.2 "Computational efficiency": "the partial forward pass of the
// Transformer backbone up to the hidden states connected to the last early
// exit").  Llama-2 pre-norm decoder layers:
//   x += W_o attn(RoPE(W_q u), RoPE(W_k u), W_v u),   u  = RMSNorm(x; g_att)
//   x += W_down(silu(W_gate u') * W_up u'),           u' = RMSNorm(x; g_mlp)
// The projections and the MLP run on the tcgen05 GEMM (gemm.cuh); this file
// holds the causal flash attention (forward and backward) and the residual
// casts; RoPE is fused into the q/k projection epilogues (gemm.cuh) and, as
// RoPE^T, into the attention backward's dq/dk stores.
//
// Attention is ~2% of a Llama-2 layer's FLOPs at T = 2048 (4 T h / 2 vs
// 2 (2 h^2 + 2 h h_kv + 3 h F) per token), so it uses warp-level mma.sync
// (m16n8k16 bf16, fp32 accumulate) in the FlashAttention-2 register layout:
// one CTA per (64-query tile, head, sequence), 4 warps x 16 query rows, K/V
// tiles of 64 keys staged in shared memory, online softmax in registers, P
// reused as the A fragments of P V.
#include <cmath>
#include "internal.cuh"

namespace ee {

// ---------------------------------------------------------------- casts
__global__ void cast_bf16_f32_kernel(const __nv_bfloat16* __restrict__ a, float* __restrict__ b,
                                     long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    b[i] = __bfloat162float(a[i]);
}
__global__ void cast_f32_bf16_kernel(const float* __restrict__ a, __nv_bfloat16* __restrict__ b,
                                     long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    b[i] = __float2bfloat16_rn(a[i]);
}
cudaError_t launch_cast_bf16_f32(const __nv_bfloat16* a, float* b, long long n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  cast_bf16_f32_kernel<<<(unsigned)min((n + 255) / 256, 65535LL * 16), 256, 0, s>>>(a, b, n);
  return cudaGetLastError();
}
cudaError_t launch_cast_f32_bf16(const float* a, __nv_bfloat16* b, long long n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  cast_f32_bf16_kernel<<<(unsigned)min((n + 255) / 256, 65535LL * 16), 256, 0, s>>>(a, b, n);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- attention
__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0,
                                               uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldmatrix_x4_trans(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}

constexpr int ATT_D = 128;   // head dim (Llama-2: 128 at every size)
constexpr int ATT_BQ = 64;   // query rows per CTA (4 warps x 16)
constexpr int ATT_BK = 64;   // keys per tile
constexpr int ATT_PAD = 8;

// o = softmax(q k^T / sqrt(d) + causal) v for each (sequence b, query head hq);
// k/v head = hq / (Hq / Hkv) (GQA).  q [N x Hq*128], k, v [N x Hkv*128],
// o [N x Hq*128], bf16; row = b * T + t.
__global__ void __launch_bounds__(128) attn_fwd_kernel(const __nv_bfloat16* __restrict__ q,
                                                       const __nv_bfloat16* __restrict__ k,
                                                       const __nv_bfloat16* __restrict__ v,
                                                       __nv_bfloat16* __restrict__ o, int T,
                                                       int Hq, int Hkv, float scale_log2,
                                                       float* __restrict__ lse2) {
  __shared__ __align__(16) __nv_bfloat16 Ks[ATT_BK][ATT_D + ATT_PAD];
  __shared__ __align__(16) __nv_bfloat16 Vs[ATT_BK][ATT_D + ATT_PAD];
  const int qt = blockIdx.x, hq = blockIdx.y, b = blockIdx.z;
  const int hk = hq / (Hq / Hkv);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, c = lane & 3;
  const long long ldq = (long long)Hq * ATT_D, ldk = (long long)Hkv * ATT_D;
  const long long qrow0 = (long long)b * T + (long long)qt * ATT_BQ + warp * 16;
  const int qpos0 = qt * ATT_BQ + warp * 16 + g;  // position of row g (row g+8: +8)

  uint32_t qa[ATT_D / 16][4];
#pragma unroll
  for (int ks = 0; ks < ATT_D / 16; ++ks) {
    const __nv_bfloat16* q0 = q + (qrow0 + g) * ldq + hq * ATT_D + ks * 16 + 2 * c;
    const __nv_bfloat16* q1 = q0 + 8 * ldq;
    qa[ks][0] = *reinterpret_cast<const uint32_t*>(q0);
    qa[ks][1] = *reinterpret_cast<const uint32_t*>(q1);
    qa[ks][2] = *reinterpret_cast<const uint32_t*>(q0 + 8);
    qa[ks][3] = *reinterpret_cast<const uint32_t*>(q1 + 8);
  }
  float oacc[ATT_D / 8][4];
#pragma unroll
  for (int nb = 0; nb < ATT_D / 8; ++nb)
#pragma unroll
    for (int e = 0; e < 4; ++e) oacc[nb][e] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

  const int nkt = qt + 1;  // causal: key tiles 0..qt (tile sizes equal)
  for (int kt = 0; kt < nkt; ++kt) {
    __syncthreads();
    const long long krow0 = (long long)b * T + (long long)kt * ATT_BK;
    for (int i = threadIdx.x; i < ATT_BK * (ATT_D / 8); i += blockDim.x) {
      const int key = i / (ATT_D / 8), ch = i % (ATT_D / 8);
      const long long off = (krow0 + key) * ldk + hk * ATT_D + ch * 8;
      *reinterpret_cast<uint4*>(&Ks[key][ch * 8]) = *reinterpret_cast<const uint4*>(k + off);
      *reinterpret_cast<uint4*>(&Vs[key][ch * 8]) = *reinterpret_cast<const uint4*>(v + off);
    }
    __syncthreads();
    // S = Q K^T (16 x 64 per warp)
    float sacc[ATT_BK / 8][4];
#pragma unroll
    for (int nb = 0; nb < ATT_BK / 8; ++nb) {
#pragma unroll
      for (int e = 0; e < 4; ++e) sacc[nb][e] = 0.f;
#pragma unroll
      for (int ks = 0; ks < ATT_D / 16; ++ks) {
        const uint32_t b0 = *reinterpret_cast<const uint32_t*>(&Ks[nb * 8 + g][ks * 16 + 2 * c]);
        const uint32_t b1 =
            *reinterpret_cast<const uint32_t*>(&Ks[nb * 8 + g][ks * 16 + 8 + 2 * c]);
        mma_bf16_16816(sacc[nb], qa[ks], b0, b1);
      }
    }
    // scale (log2 domain), causal mask on the diagonal tile, online softmax
    float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
    for (int nb = 0; nb < ATT_BK / 8; ++nb) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int kpos = kt * ATT_BK + nb * 8 + 2 * c + (e & 1);
        const int qpos = qpos0 + (e >= 2 ? 8 : 0);
        float x = sacc[nb][e] * scale_log2;
        if (kt == qt && kpos > qpos) x = -INFINITY;
        sacc[nb][e] = x;
      }
      mx0 = fmaxf(mx0, fmaxf(sacc[nb][0], sacc[nb][1]));
      mx1 = fmaxf(mx1, fmaxf(sacc[nb][2], sacc[nb][3]));
    }
#pragma unroll
    for (int sh = 1; sh <= 2; sh <<= 1) {
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, sh));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, sh));
    }
    const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);  // finite: diagonal always valid
    const float al0 = exp2f(m0 - mn0), al1 = exp2f(m1 - mn1);
    m0 = mn0;
    m1 = mn1;
    l0 *= al0;
    l1 *= al1;
#pragma unroll
    for (int nb = 0; nb < ATT_D / 8; ++nb) {
      oacc[nb][0] *= al0;
      oacc[nb][1] *= al0;
      oacc[nb][2] *= al1;
      oacc[nb][3] *= al1;
    }
    uint32_t pa[ATT_BK / 16][4];
#pragma unroll
    for (int nb = 0; nb < ATT_BK / 8; ++nb) {
      const float p0 = exp2f(sacc[nb][0] - m0), p1 = exp2f(sacc[nb][1] - m0);
      const float p2 = exp2f(sacc[nb][2] - m1), p3 = exp2f(sacc[nb][3] - m1);
      l0 += p0 + p1;
      l1 += p2 + p3;
      const int kk = nb >> 1, hi = nb & 1;
      pa[kk][hi ? 2 : 0] = pack_bf16(p0, p1);
      pa[kk][hi ? 3 : 1] = pack_bf16(p2, p3);
    }
    // O += P V: B fragments of V (k = key, n = d) via ldmatrix.trans
#pragma unroll
    for (int kk = 0; kk < ATT_BK / 16; ++kk) {
#pragma unroll
      for (int nb = 0; nb < ATT_D / 8; nb += 2) {
        // matrices: (keys kk*16+0..7, d nb*8..), (keys +8..15, d nb*8..),
        //           (keys kk*16+0..7, d (nb+1)*8..), (keys +8..15, d (nb+1)*8..)
        const int mi = lane >> 3, r = lane & 7;
        const int key = kk * 16 + (mi & 1) * 8 + r;
        const int dcol = (nb + (mi >> 1)) * 8;
        uint32_t bv[4];
        ldmatrix_x4_trans(bv, &Vs[key][dcol]);
        mma_bf16_16816(oacc[nb], pa[kk], bv[0], bv[1]);
        mma_bf16_16816(oacc[nb + 1], pa[kk], bv[2], bv[3]);
      }
    }
  }
#pragma unroll
  for (int sh = 1; sh <= 2; sh <<= 1) {
    l0 += __shfl_xor_sync(0xffffffffu, l0, sh);
    l1 += __shfl_xor_sync(0xffffffffu, l1, sh);
  }
  const float i0 = 1.0f / l0, i1 = 1.0f / l1;
  if (lse2 != nullptr && c == 0) {  // row statistics for the backward: log2-domain lse
    lse2[(qrow0 + g) * Hq + hq] = m0 + log2f(l0);
    lse2[(qrow0 + g + 8) * Hq + hq] = m1 + log2f(l1);
  }
  __nv_bfloat16* o0 = o + (qrow0 + g) * ldq + hq * ATT_D + 2 * c;
  __nv_bfloat16* o1 = o0 + 8 * ldq;
#pragma unroll
  for (int nb = 0; nb < ATT_D / 8; ++nb) {
    *reinterpret_cast<uint32_t*>(o0 + nb * 8) = pack_bf16(oacc[nb][0] * i0, oacc[nb][1] * i0);
    *reinterpret_cast<uint32_t*>(o1 + nb * 8) = pack_bf16(oacc[nb][2] * i1, oacc[nb][3] * i1);
  }
}

cudaError_t launch_attn_fwd(const __nv_bfloat16* q, const __nv_bfloat16* k, const __nv_bfloat16* v,
                            __nv_bfloat16* o, long long N, int T, int Hq, int Hkv, float* lse2,
                            cudaStream_t s) {
  if (N == 0) return cudaSuccess;
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)ATT_D);
  dim3 grid(T / ATT_BQ, Hq, (unsigned)(N / T));
  attn_fwd_kernel<<<grid, 128, 0, s>>>(q, k, v, o, T, Hq, Hkv, scale_log2, lse2);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- attention backward
// FlashAttention-2 backward, split deterministically into
//   attn_bwd_dkdv: one CTA per (64-key tile, kv head, sequence), looping over the
//     query heads of its GQA group and the causal query tiles; dK, dV stay in
//     registers (no atomics);
//   attn_bwd_dq:   one CTA per (64-query tile, query head, sequence), looping
//     over the causal key tiles.
// With lse2 = log2-domain row statistics of the forward and
// Dv = rowsum(dO * O):  P = exp2(s S - lse2),  dP = dO V^T,
//   dS = P (dP - Dv),  dQ = c dS K,  dK = c dS^T Q,  dV = P^T dO  (c = 1/sqrt(d)).
__global__ void attn_bwd_dot_kernel(const __nv_bfloat16* __restrict__ o,
                                    const __nv_bfloat16* __restrict__ dout, float* __restrict__ Dv,
                                    long long rows_heads) {
  // one warp per (row, head): 128 elements
  const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= rows_heads) return;
  const uint2 a = *reinterpret_cast<const uint2*>(o + w * 128 + lane * 4);
  const uint2 b = *reinterpret_cast<const uint2*>(dout + w * 128 + lane * 4);
  float acc = bf16lo(a.x) * bf16lo(b.x) + bf16hi(a.x) * bf16hi(b.x) + bf16lo(a.y) * bf16lo(b.y) +
              bf16hi(a.y) * bf16hi(b.y);
#pragma unroll
  for (int sh = 16; sh > 0; sh >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, sh);
  if (lane == 0) Dv[w] = acc;
}

// RoPE^T (rotation by -angle) applied in fp32 to an accumulator fragment
// acc[nb][e] = row (pos0 + (e >= 2 ? 8 : 0)), column nb * 8 + 2c + (e & 1) of a
// 128-wide head: column i (nb < 8) pairs with i + 64 (nb + 8) in this thread.
__device__ __forceinline__ void rope_t_frag(float (&acc)[ATT_D / 8][4], int pos0, int c,
                                            float theta) {
#pragma unroll
  for (int nb = 0; nb < ATT_D / 16; ++nb) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int i = nb * 8 + 2 * c + (e & 1);
      const float pos = (float)(pos0 + (e >= 2 ? 8 : 0));
      const float inv = powf(theta, -2.0f * (float)i / 128.0f);
      float sn, cs;
      sincosf(pos * inv, &sn, &cs);
      const float a = acc[nb][e], b = acc[nb + 8][e];
      acc[nb][e] = a * cs + b * sn;
      acc[nb + 8][e] = b * cs - a * sn;
    }
  }
}

__device__ __forceinline__ void ldmatrix_x4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}

__global__ void __launch_bounds__(128) attn_bwd_dkdv_kernel(
    const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k,
    const __nv_bfloat16* __restrict__ v, const __nv_bfloat16* __restrict__ dout,
    const float* __restrict__ lse2, const float* __restrict__ Dv, __nv_bfloat16* __restrict__ dk,
    __nv_bfloat16* __restrict__ dv, int T, int Hq, int Hkv, float scale_log2, float scale,
    float rope_theta) {
  __shared__ __align__(16) __nv_bfloat16 Qs[ATT_BQ][ATT_D + ATT_PAD];
  __shared__ __align__(16) __nv_bfloat16 Os[ATT_BQ][ATT_D + ATT_PAD];  // dO tile
  __shared__ float Ls[ATT_BQ], Ds[ATT_BQ];
  const int kt = blockIdx.x, hk = blockIdx.y, b = blockIdx.z;
  const int grp = Hq / Hkv;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, c = lane & 3;
  const long long ldq = (long long)Hq * ATT_D, ldk = (long long)Hkv * ATT_D;
  const long long krow0 = (long long)b * T + (long long)kt * ATT_BK + warp * 16;  // this warp's keys
  const int kpos0 = kt * ATT_BK + warp * 16 + g;

  // K_w and V_w (16 keys x 128 d) as A fragments
  uint32_t ka[ATT_D / 16][4], va[ATT_D / 16][4];
#pragma unroll
  for (int ks = 0; ks < ATT_D / 16; ++ks) {
    const __nv_bfloat16* k0 = k + (krow0 + g) * ldk + hk * ATT_D + ks * 16 + 2 * c;
    const __nv_bfloat16* v0 = v + (krow0 + g) * ldk + hk * ATT_D + ks * 16 + 2 * c;
    ka[ks][0] = *reinterpret_cast<const uint32_t*>(k0);
    ka[ks][1] = *reinterpret_cast<const uint32_t*>(k0 + 8 * ldk);
    ka[ks][2] = *reinterpret_cast<const uint32_t*>(k0 + 8);
    ka[ks][3] = *reinterpret_cast<const uint32_t*>(k0 + 8 * ldk + 8);
    va[ks][0] = *reinterpret_cast<const uint32_t*>(v0);
    va[ks][1] = *reinterpret_cast<const uint32_t*>(v0 + 8 * ldk);
    va[ks][2] = *reinterpret_cast<const uint32_t*>(v0 + 8);
    va[ks][3] = *reinterpret_cast<const uint32_t*>(v0 + 8 * ldk + 8);
  }
  float dka[ATT_D / 8][4], dva[ATT_D / 8][4];
#pragma unroll
  for (int nb = 0; nb < ATT_D / 8; ++nb)
#pragma unroll
    for (int e = 0; e < 4; ++e) dka[nb][e] = dva[nb][e] = 0.f;

  const int nqt = T / ATT_BQ;
  for (int hh = 0; hh < grp; ++hh) {
    const int hq = hk * grp + hh;
    for (int qt = kt; qt < nqt; ++qt) {  // causal: queries at or after this key tile
      __syncthreads();
      const long long qrow0 = (long long)b * T + (long long)qt * ATT_BQ;
      for (int i = threadIdx.x; i < ATT_BQ * (ATT_D / 8); i += blockDim.x) {
        const int r = i / (ATT_D / 8), ch = i % (ATT_D / 8);
        const long long off = (qrow0 + r) * ldq + hq * ATT_D + ch * 8;
        *reinterpret_cast<uint4*>(&Qs[r][ch * 8]) = *reinterpret_cast<const uint4*>(q + off);
        *reinterpret_cast<uint4*>(&Os[r][ch * 8]) = *reinterpret_cast<const uint4*>(dout + off);
      }
      if (threadIdx.x < ATT_BQ) {
        Ls[threadIdx.x] = lse2[(qrow0 + threadIdx.x) * Hq + hq];
        Ds[threadIdx.x] = Dv[(qrow0 + threadIdx.x) * Hq + hq];
      }
      __syncthreads();
      // S^T = K_w Q^T (16 keys x 64 queries);  dP^T = V_w dO^T
      float st[ATT_BQ / 8][4], dpt[ATT_BQ / 8][4];
#pragma unroll
      for (int nb = 0; nb < ATT_BQ / 8; ++nb) {
#pragma unroll
        for (int e = 0; e < 4; ++e) st[nb][e] = dpt[nb][e] = 0.f;
#pragma unroll
        for (int ks = 0; ks < ATT_D / 16; ++ks) {
          const uint32_t b0 = *reinterpret_cast<const uint32_t*>(&Qs[nb * 8 + g][ks * 16 + 2 * c]);
          const uint32_t b1 =
              *reinterpret_cast<const uint32_t*>(&Qs[nb * 8 + g][ks * 16 + 8 + 2 * c]);
          mma_bf16_16816(st[nb], ka[ks], b0, b1);
          const uint32_t e0 = *reinterpret_cast<const uint32_t*>(&Os[nb * 8 + g][ks * 16 + 2 * c]);
          const uint32_t e1 =
              *reinterpret_cast<const uint32_t*>(&Os[nb * 8 + g][ks * 16 + 8 + 2 * c]);
          mma_bf16_16816(dpt[nb], va[ks], e0, e1);
        }
      }
      // P^T and dS^T (rows = keys g / g+8, cols = queries nb*8 + 2c (+1))
      uint32_t pa[ATT_BQ / 16][4], sa[ATT_BQ / 16][4];
#pragma unroll
      for (int nb = 0; nb < ATT_BQ / 8; ++nb) {
        float p[4], d[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int qi = nb * 8 + 2 * c + (e & 1);
          const int qpos = qt * ATT_BQ + qi;
          const int kpos = kpos0 + (e >= 2 ? 8 : 0);
          float pv = exp2f(st[nb][e] * scale_log2 - Ls[qi]);
          if (qt == kt && kpos > qpos) pv = 0.f;
          p[e] = pv;
          d[e] = pv * (dpt[nb][e] - Ds[qi]);
        }
        const int kk = nb >> 1, hi = nb & 1;
        pa[kk][hi ? 2 : 0] = pack_bf16(p[0], p[1]);
        pa[kk][hi ? 3 : 1] = pack_bf16(p[2], p[3]);
        sa[kk][hi ? 2 : 0] = pack_bf16(d[0], d[1]);
        sa[kk][hi ? 3 : 1] = pack_bf16(d[2], d[3]);
      }
      // dV += P^T dO ; dK += dS^T Q   (B = [q][d] tiles via ldmatrix.trans)
#pragma unroll
      for (int kk = 0; kk < ATT_BQ / 16; ++kk) {
#pragma unroll
        for (int nb = 0; nb < ATT_D / 8; nb += 2) {
          const int mi = lane >> 3, r = lane & 7;
          const int qi = kk * 16 + (mi & 1) * 8 + r;
          const int dcol = (nb + (mi >> 1)) * 8;
          uint32_t bo[4], bq[4];
          ldmatrix_x4_trans(bo, &Os[qi][dcol]);
          ldmatrix_x4_trans(bq, &Qs[qi][dcol]);
          mma_bf16_16816(dva[nb], pa[kk], bo[0], bo[1]);
          mma_bf16_16816(dva[nb + 1], pa[kk], bo[2], bo[3]);
          mma_bf16_16816(dka[nb], sa[kk], bq[0], bq[1]);
          mma_bf16_16816(dka[nb + 1], sa[kk], bq[2], bq[3]);
        }
      }
    }
  }
  if (rope_theta > 0.f) rope_t_frag(dka, kpos0, c, rope_theta);
  __nv_bfloat16* k0 = dk + (krow0 + g) * ldk + hk * ATT_D + 2 * c;
  __nv_bfloat16* v0 = dv + (krow0 + g) * ldk + hk * ATT_D + 2 * c;
#pragma unroll
  for (int nb = 0; nb < ATT_D / 8; ++nb) {
    *reinterpret_cast<uint32_t*>(k0 + nb * 8) = pack_bf16(dka[nb][0] * scale, dka[nb][1] * scale);
    *reinterpret_cast<uint32_t*>(k0 + 8 * ldk + nb * 8) =
        pack_bf16(dka[nb][2] * scale, dka[nb][3] * scale);
    *reinterpret_cast<uint32_t*>(v0 + nb * 8) = pack_bf16(dva[nb][0], dva[nb][1]);
    *reinterpret_cast<uint32_t*>(v0 + 8 * ldk + nb * 8) = pack_bf16(dva[nb][2], dva[nb][3]);
  }
}

__global__ void __launch_bounds__(128) attn_bwd_dq_kernel(
    const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k,
    const __nv_bfloat16* __restrict__ v, const __nv_bfloat16* __restrict__ dout,
    const float* __restrict__ lse2, const float* __restrict__ Dv, __nv_bfloat16* __restrict__ dq,
    int T, int Hq, int Hkv, float scale_log2, float scale, float rope_theta) {
  __shared__ __align__(16) __nv_bfloat16 Ks[ATT_BK][ATT_D + ATT_PAD];
  __shared__ __align__(16) __nv_bfloat16 Vs[ATT_BK][ATT_D + ATT_PAD];
  const int qt = blockIdx.x, hq = blockIdx.y, b = blockIdx.z;
  const int hk = hq / (Hq / Hkv);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, c = lane & 3;
  const long long ldq = (long long)Hq * ATT_D, ldk = (long long)Hkv * ATT_D;
  const long long qrow0 = (long long)b * T + (long long)qt * ATT_BQ + warp * 16;
  const int qpos0 = qt * ATT_BQ + warp * 16 + g;
  uint32_t qa[ATT_D / 16][4], oa[ATT_D / 16][4];
#pragma unroll
  for (int ks = 0; ks < ATT_D / 16; ++ks) {
    const __nv_bfloat16* q0 = q + (qrow0 + g) * ldq + hq * ATT_D + ks * 16 + 2 * c;
    const __nv_bfloat16* o0 = dout + (qrow0 + g) * ldq + hq * ATT_D + ks * 16 + 2 * c;
    qa[ks][0] = *reinterpret_cast<const uint32_t*>(q0);
    qa[ks][1] = *reinterpret_cast<const uint32_t*>(q0 + 8 * ldq);
    qa[ks][2] = *reinterpret_cast<const uint32_t*>(q0 + 8);
    qa[ks][3] = *reinterpret_cast<const uint32_t*>(q0 + 8 * ldq + 8);
    oa[ks][0] = *reinterpret_cast<const uint32_t*>(o0);
    oa[ks][1] = *reinterpret_cast<const uint32_t*>(o0 + 8 * ldq);
    oa[ks][2] = *reinterpret_cast<const uint32_t*>(o0 + 8);
    oa[ks][3] = *reinterpret_cast<const uint32_t*>(o0 + 8 * ldq + 8);
  }
  const float l0 = lse2[(qrow0 + g) * Hq + hq], l1 = lse2[(qrow0 + g + 8) * Hq + hq];
  const float d0 = Dv[(qrow0 + g) * Hq + hq], d1 = Dv[(qrow0 + g + 8) * Hq + hq];
  float dqa[ATT_D / 8][4];
#pragma unroll
  for (int nb = 0; nb < ATT_D / 8; ++nb)
#pragma unroll
    for (int e = 0; e < 4; ++e) dqa[nb][e] = 0.f;
  for (int kt = 0; kt <= qt; ++kt) {
    __syncthreads();
    const long long krow0 = (long long)b * T + (long long)kt * ATT_BK;
    for (int i = threadIdx.x; i < ATT_BK * (ATT_D / 8); i += blockDim.x) {
      const int key = i / (ATT_D / 8), ch = i % (ATT_D / 8);
      const long long off = (krow0 + key) * ldk + hk * ATT_D + ch * 8;
      *reinterpret_cast<uint4*>(&Ks[key][ch * 8]) = *reinterpret_cast<const uint4*>(k + off);
      *reinterpret_cast<uint4*>(&Vs[key][ch * 8]) = *reinterpret_cast<const uint4*>(v + off);
    }
    __syncthreads();
    float sacc[ATT_BK / 8][4], dpa[ATT_BK / 8][4];
#pragma unroll
    for (int nb = 0; nb < ATT_BK / 8; ++nb) {
#pragma unroll
      for (int e = 0; e < 4; ++e) sacc[nb][e] = dpa[nb][e] = 0.f;
#pragma unroll
      for (int ks = 0; ks < ATT_D / 16; ++ks) {
        const uint32_t b0 = *reinterpret_cast<const uint32_t*>(&Ks[nb * 8 + g][ks * 16 + 2 * c]);
        const uint32_t b1 =
            *reinterpret_cast<const uint32_t*>(&Ks[nb * 8 + g][ks * 16 + 8 + 2 * c]);
        mma_bf16_16816(sacc[nb], qa[ks], b0, b1);
        const uint32_t e0 = *reinterpret_cast<const uint32_t*>(&Vs[nb * 8 + g][ks * 16 + 2 * c]);
        const uint32_t e1 =
            *reinterpret_cast<const uint32_t*>(&Vs[nb * 8 + g][ks * 16 + 8 + 2 * c]);
        mma_bf16_16816(dpa[nb], oa[ks], e0, e1);
      }
    }
    uint32_t sa[ATT_BK / 16][4];
#pragma unroll
    for (int nb = 0; nb < ATT_BK / 8; ++nb) {
      float ds[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int kpos = kt * ATT_BK + nb * 8 + 2 * c + (e & 1);
        const int qpos = qpos0 + (e >= 2 ? 8 : 0);
        float pv = exp2f(sacc[nb][e] * scale_log2 - (e >= 2 ? l1 : l0));
        if (kt == qt && kpos > qpos) pv = 0.f;
        ds[e] = pv * (dpa[nb][e] - (e >= 2 ? d1 : d0));
      }
      const int kk = nb >> 1, hi = nb & 1;
      sa[kk][hi ? 2 : 0] = pack_bf16(ds[0], ds[1]);
      sa[kk][hi ? 3 : 1] = pack_bf16(ds[2], ds[3]);
    }
    // dQ += dS K  (B[k = key][n = d] = K[key][d] via ldmatrix.trans)
#pragma unroll
    for (int kk = 0; kk < ATT_BK / 16; ++kk) {
#pragma unroll
      for (int nb = 0; nb < ATT_D / 8; nb += 2) {
        const int mi = lane >> 3, r = lane & 7;
        const int key = kk * 16 + (mi & 1) * 8 + r;
        const int dcol = (nb + (mi >> 1)) * 8;
        uint32_t bk[4];
        ldmatrix_x4_trans(bk, &Ks[key][dcol]);
        mma_bf16_16816(dqa[nb], sa[kk], bk[0], bk[1]);
        mma_bf16_16816(dqa[nb + 1], sa[kk], bk[2], bk[3]);
      }
    }
  }
  if (rope_theta > 0.f) rope_t_frag(dqa, qpos0, c, rope_theta);
  __nv_bfloat16* q0 = dq + (qrow0 + g) * ldq + hq * ATT_D + 2 * c;
#pragma unroll
  for (int nb = 0; nb < ATT_D / 8; ++nb) {
    *reinterpret_cast<uint32_t*>(q0 + nb * 8) = pack_bf16(dqa[nb][0] * scale, dqa[nb][1] * scale);
    *reinterpret_cast<uint32_t*>(q0 + 8 * ldq + nb * 8) =
        pack_bf16(dqa[nb][2] * scale, dqa[nb][3] * scale);
  }
}

cudaError_t launch_attn_bwd(const __nv_bfloat16* q, const __nv_bfloat16* k, const __nv_bfloat16* v,
                            const __nv_bfloat16* o, const __nv_bfloat16* dout, const float* lse2,
                            float* Dv, __nv_bfloat16* dq, __nv_bfloat16* dk, __nv_bfloat16* dv,
                            long long N, int T, int Hq, int Hkv, float rope_theta,
                            cudaStream_t s, bool tc, const float2* rope_tab) {
  if (N == 0) return cudaSuccess;
  const float scale = 1.0f / sqrtf((float)ATT_D);
  const float scale_log2 = 1.4426950408889634f * scale;
  const long long rh = N * Hq;
  attn_bwd_dot_kernel<<<(unsigned)((rh * 32 + 255) / 256), 256, 0, s>>>(o, dout, Dv, rh);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (tc)
    return launch_attn_bwd_tc(q, k, v, dout, lse2, Dv, dq, dk, dv, N, T, Hq, Hkv, rope_theta, s,
                              rope_tab);
  dim3 g1(T / ATT_BK, Hkv, (unsigned)(N / T));
  attn_bwd_dkdv_kernel<<<g1, 128, 0, s>>>(q, k, v, dout, lse2, Dv, dk, dv, T, Hq, Hkv, scale_log2,
                                          scale, rope_theta);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  dim3 g2(T / ATT_BQ, Hq, (unsigned)(N / T));
  attn_bwd_dq_kernel<<<g2, 128, 0, s>>>(q, k, v, dout, lse2, Dv, dq, T, Hq, Hkv, scale_log2, scale,
                                        rope_theta);
  return cudaGetLastError();
}


}  // namespace ee
