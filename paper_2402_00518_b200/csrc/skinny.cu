// skinny.cu -- decode-shape exit heads for the confidence-based early-exit
// decision at inference (NEXT #4): M <= 16 tokens per call, so the
// exit head is a stream over its weights (arithmetic intensity <= 16 flop/B,
// HBM-bound) and the training GEMM's 256-wide tiles would leave most SMs idle
// (W_down: 32 tiles).  One warp per 8 weight rows, 128-bit streaming loads
// along K, warp-level bf16 MMA with fp32 accumulation; 32 columns per CTA.
// Epilogues: SwiGLU (gate and up rows of the same index in one warp),
// residual add (fp32 out), and online-softmax statistics per 32-column block
// (the same [block x token] partials layout ce_finalize reads).
#include <cfloat>
#include <climits>
#include "internal.cuh"

namespace ee {

namespace {
constexpr int SK_WARPS = 4, SK_RW = 8, SK_COLS = SK_WARPS * SK_RW;  // 32 weight rows per CTA
constexpr int SK_KS = 4;       // K split over 4 warps per row group (bytes in flight per CTA)
constexpr int SK_UNROLL = 4;   // 16-byte loads in flight per thread and row

__device__ __forceinline__ uint4 ld_stream(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// One 32-wide K chunk: thread (g, c) holds 8 consecutive k of W row g and of
// tokens g (x0) and g + 8 (x1) (the dot product is order-independent, so the
// MMA's k positions 2c, 2c+1 | 2c+8, 2c+9 of step s are mapped to
// k = 8c + 4s + {0,1} | {2,3}).
__device__ __forceinline__ void mma_chunk(float (&d)[4], const uint4& x0, const uint4& x1,
                                          const uint4& w) {
  mma16816(d, x0.x, x1.x, x0.y, x1.y, w.x, w.y);
  mma16816(d, x0.z, x1.z, x0.w, x1.w, w.z, w.w);
}
}  // namespace

// out[m][n] = sum_k x[m][k] W[n][k], m < M <= 8 tokens: one warp per 8 weight
// rows; warp-level bf16 MMA (m16n8k16, fp32 accumulate; tokens padded to 16)
// so the kernel streams W at HBM speed with one 128-bit load per 32 k.
template <int M, int MODE>
__global__ void __launch_bounds__(32 * SK_WARPS * SK_KS) skinny_kernel(SkinnyArgs a) {
  __shared__ float s_log[16][SK_COLS];
  __shared__ float4 s_red[SK_KS - 1][SK_WARPS][2][32];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int warp = wid % SK_WARPS, ks = wid / SK_WARPS;   // row group, K slice
  const int g = lane >> 2, c = lane & 3;
  const int n0 = blockIdx.x * SK_COLS + warp * SK_RW;
  const int nrow = min(n0 + g, a.N - 1);
  const __nv_bfloat16* w0 = a.W0 + (long long)nrow * a.K + 8 * c;
  const __nv_bfloat16* w1 = (MODE == SK_SWIGLU) ? a.W1 + (long long)nrow * a.K + 8 * c : nullptr;
  const bool tok = g < M, tok1 = M > 8 && g + 8 < M;   // tokens g and g + 8
  const __nv_bfloat16* xr = a.x + (long long)(tok ? g : 0) * a.ldx + 8 * c;
  const __nv_bfloat16* xr1 = a.x + (long long)(tok1 ? g + 8 : 0) * a.ldx + 8 * c;
  float d0[4] = {0.f, 0.f, 0.f, 0.f}, d1[4] = {0.f, 0.f, 0.f, 0.f};
  const uint4 zero = make_uint4(0u, 0u, 0u, 0u);
  // K slices interleaved in 32 * SK_UNROLL-wide blocks
  constexpr int KB = 32 * SK_UNROLL;
  int k = ks * KB;
  // software-pipelined: block i + 1's loads are issued before block i's MMAs
  // (registers carried across iterations), so ptxas cannot interleave loads
  // and uses and 2 x SK_UNROLL weight loads per thread stay in flight
  uint4 wv[SK_UNROLL], uv[SK_UNROLL], xv[SK_UNROLL], xw[SK_UNROLL];
  auto load_block = [&](int kk, uint4 (&w)[SK_UNROLL], uint4 (&u1)[SK_UNROLL],
                        uint4 (&x0)[SK_UNROLL], uint4 (&x1)[SK_UNROLL]) {
#pragma unroll
    for (int u = 0; u < SK_UNROLL; ++u) {
      w[u] = ld_stream(w0 + kk + 32 * u);
      if (MODE == SK_SWIGLU) u1[u] = ld_stream(w1 + kk + 32 * u);
      x0[u] = tok ? __ldg(reinterpret_cast<const uint4*>(xr + kk + 32 * u)) : zero;
      x1[u] = tok1 ? __ldg(reinterpret_cast<const uint4*>(xr1 + kk + 32 * u)) : zero;
    }
  };
  if (k + KB <= a.K) load_block(k, wv, uv, xv, xw);
  for (; k + KB <= a.K; k += SK_KS * KB) {
    uint4 wn[SK_UNROLL], un[SK_UNROLL], xn[SK_UNROLL], xm[SK_UNROLL];
    const bool more = k + SK_KS * KB + KB <= a.K;
    if (more) load_block(k + SK_KS * KB, wn, un, xn, xm);
#pragma unroll
    for (int u = 0; u < SK_UNROLL; ++u) {
      mma_chunk(d0, xv[u], xw[u], wv[u]);
      if (MODE == SK_SWIGLU) mma_chunk(d1, xv[u], xw[u], uv[u]);
    }
    if (more) {
#pragma unroll
      for (int u = 0; u < SK_UNROLL; ++u) {
        wv[u] = wn[u];
        if (MODE == SK_SWIGLU) uv[u] = un[u];
        xv[u] = xn[u];
        xw[u] = xm[u];
      }
    }
  }
  if (k < a.K) {  // this slice's partial last block (K % 8 == 0; zeros past K)
    for (int u = 0; u < SK_UNROLL; ++u) {
      const int kk = k + 32 * u;
      const bool in = kk + 8 * c < a.K;
      const uint4 wv = in ? ld_stream(w0 + kk) : zero;
      const uint4 xv = (in && tok) ? __ldg(reinterpret_cast<const uint4*>(xr + kk)) : zero;
      const uint4 xw = (in && tok1) ? __ldg(reinterpret_cast<const uint4*>(xr1 + kk)) : zero;
      mma_chunk(d0, xv, xw, wv);
      if (MODE == SK_SWIGLU) {
        const uint4 uv = in ? ld_stream(w1 + kk) : zero;
        mma_chunk(d1, xv, xw, uv);
      }
    }
  }
  // reduce the K slices into slice 0 (fixed order: deterministic)
  if (ks > 0) {
    s_red[ks - 1][warp][0][lane] = make_float4(d0[0], d0[1], d0[2], d0[3]);
    if (MODE == SK_SWIGLU) s_red[ks - 1][warp][1][lane] = make_float4(d1[0], d1[1], d1[2], d1[3]);
  }
  __syncthreads();
  if (ks > 0) return;
#pragma unroll
  for (int q = 0; q < SK_KS - 1; ++q) {
    const float4 p = s_red[q][warp][0][lane];
    d0[0] += p.x; d0[1] += p.y; d0[2] += p.z; d0[3] += p.w;
    if (MODE == SK_SWIGLU) {
      const float4 r = s_red[q][warp][1][lane];
      d1[0] += r.x; d1[1] += r.y; d1[2] += r.z; d1[3] += r.w;
    }
  }
  // d[0], d[1] = out[token g][n0 + 2c (+1)]; d[2], d[3] = out[token g + 8][...]
  const int na = n0 + 2 * c;
  if constexpr (MODE == SK_CE) {
    if (tok) {
      s_log[g][warp * SK_RW + 2 * c] = na < a.N ? d0[0] : -INFINITY;
      s_log[g][warp * SK_RW + 2 * c + 1] = na + 1 < a.N ? d0[1] : -INFINITY;
    }
    if (tok1) {
      s_log[g + 8][warp * SK_RW + 2 * c] = na < a.N ? d0[2] : -INFINITY;
      s_log[g + 8][warp * SK_RW + 2 * c + 1] = na + 1 < a.N ? d0[3] : -INFINITY;
    }
    asm volatile("bar.sync 1, %0;" ::"n"(32 * SK_WARPS) : "memory");  // the K-slice-0 warps
    for (int m = warp; m < M; m += SK_WARPS) {  // token m's statistics over the 32 columns
      const float v = s_log[m][lane];
      float mx = v;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      float se = v == -INFINITY ? 0.f : __expf(v - mx);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
      const unsigned ball = __ballot_sync(0xffffffffu, v == mx);
      if (lane == 0) {
        const long long j = blockIdx.x;
        a.pm[j * M + m] = mx;
        a.ps[j * M + m] = se;
        a.pi[j * M + m] = a.vocab_begin + blockIdx.x * SK_COLS + (__ffs(ball) - 1);
      }
    }
  } else {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int tk = g + (e >= 2 ? 8 : 0);
      const int n = na + (e & 1);
      if (!(e >= 2 ? tok1 : tok) || n >= a.N) continue;
      const long long o = (long long)tk * a.ldo + n;
      if constexpr (MODE == SK_SWIGLU) {
        const float v = d0[e], u = d1[e];
        a.outb[o] = __float2bfloat16_rn(__fdividef(v, 1.0f + __expf(-v)) * u);
      } else if constexpr (MODE == SK_RESID) {
        a.out[o] = d0[e] + __bfloat162float(a.resid[(long long)tk * a.ldr + n]);
      } else {
        a.out[o] = d0[e];
      }
    }
  }
}

template <int MODE>
static cudaError_t launch_m(const SkinnyArgs& a, int M, cudaStream_t s) {
  const unsigned grid = (unsigned)((a.N + SK_COLS - 1) / SK_COLS);
  switch (M) {
#define EE_SK(m) case m: skinny_kernel<m, MODE><<<grid, 32 * SK_WARPS * SK_KS, 0, s>>>(a); break;
    EE_SK(1) EE_SK(2) EE_SK(3) EE_SK(4) EE_SK(5) EE_SK(6) EE_SK(7) EE_SK(8)
    EE_SK(9) EE_SK(10) EE_SK(11) EE_SK(12) EE_SK(13) EE_SK(14) EE_SK(15) EE_SK(16)
#undef EE_SK
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

int skinny_blocks(int N) { return (N + SK_COLS - 1) / SK_COLS; }

// Inference finalize for the decode path: one 256-thread block per token over
// the nb vocab-block partials [nb x M] (the training finalize walks them with
// one thread per token, which is latency-bound at nb = V/32 and M <= 8).
// lse = m + ln s; conf = 1/s (max softmax probability); argmax = the
// lowest vocab index attaining the max (A9).
__global__ void __launch_bounds__(256) infer_finalize_wide_kernel(
    const float* __restrict__ pm, const float* __restrict__ ps, const int32_t* __restrict__ pi,
    int nb, int M, float* __restrict__ lse, int32_t* __restrict__ argmax, float* __restrict__ conf) {
  __shared__ float s_m[8], s_s[8];   // 8 warps
  __shared__ int s_i[8];
  const int t = blockIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float m = -INFINITY;
  for (int j = threadIdx.x; j < nb; j += blockDim.x) m = fmaxf(m, pm[(long long)j * M + t]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) s_m[w] = m;
  __syncthreads();
  m = s_m[0];
#pragma unroll
  for (int q = 1; q < 8; ++q) m = fmaxf(m, s_m[q]);
  float sum = 0.f;
  int am = INT_MAX;
  for (int j = threadIdx.x; j < nb; j += blockDim.x) {
    const float mj = pm[(long long)j * M + t];
    sum += ps[(long long)j * M + t] * __expf(mj - m);
    if (mj == m) am = min(am, pi[(long long)j * M + t]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sum += __shfl_xor_sync(0xffffffffu, sum, o);
    am = min(am, __shfl_xor_sync(0xffffffffu, am, o));
  }
  __syncthreads();
  if (lane == 0) {
    s_s[w] = sum;
    s_i[w] = am;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float ssum = 0.f;
    int a_ = INT_MAX;
    for (int q = 0; q < 8; ++q) {
      ssum += s_s[q];
      a_ = min(a_, s_i[q]);
    }
    if (lse) lse[t] = m + logf(ssum);
    if (argmax) argmax[t] = a_;
    if (conf) conf[t] = 1.0f / ssum;
  }
}

cudaError_t launch_infer_finalize_wide(const float* pm, const float* ps, const int32_t* pi, int nb,
                                       int M, float* lse, int32_t* argmax, float* conf,
                                       cudaStream_t s) {
  if (M == 0) return cudaSuccess;
  infer_finalize_wide_kernel<<<M, 256, 0, s>>>(pm, ps, pi, nb, M, lse, argmax, conf);
  return cudaGetLastError();
}

cudaError_t launch_skinny(int mode, const SkinnyArgs& a, int M, cudaStream_t s) {
  if (M < 1 || M > SKINNY_MAX_M || a.K % 8 != 0) return cudaErrorInvalidValue;
  switch (mode) {
    case SK_F32: return launch_m<SK_F32>(a, M, s);
    case SK_RESID: return launch_m<SK_RESID>(a, M, s);
    case SK_SWIGLU: return launch_m<SK_SWIGLU>(a, M, s);
    case SK_CE: return launch_m<SK_CE>(a, M, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace ee
