// skinny.cu -- decode-shape exit heads for the confidence-based early-exit
// decision at inference (NEXT #4): M <= 16 tokens per call, so the
// exit head is a stream over its weights (arithmetic intensity <= 16 flop/B,
// HBM-bound) and the training GEMM's 256-wide tiles would leave most SMs idle
// (W_down: 32 tiles).
//
// Design (round 2, replacing a register-fed kernel whose gate|up instantiation
// spilled for M > 8 and whose 1-CTA-per-SM grids of 256 / 1000 row blocks left
// partial last waves; profiles/r02w_decode_launches.md):
//   * TMA-fed: warp 4 streams two 32-row x 256-k weight tiles per stage (SwiGLU:
//     gate and up rows of the same index; the other modes: row blocks rb and
//     rb + half of the one matrix) and the matching [M x 256] slice of
//     the activations through a 5-10 stage shared-memory ring (128B swizzle,
//     ~200 KB in flight per SM) -- no registers hold loads in flight.
//   * Four consumer warps, 8 weight rows each: warp-level bf16 MMA (m16n8k16,
//     fp32 accumulate, tokens padded to 16) from conflict-free swizzled smem.
//   * Stream-K over (row block, k chunk) units: one persistent CTA per SM
//     takes an equal contiguous range, so every SM streams the same number of
//     bytes.  A row block split between CTAs is finished by the CTA holding its
//     first chunk; the later CTAs publish their partial sums (fp32, in a
//     device pool) at the very start of their ranges and the finisher adds them
//     in CTA order -- deterministic, and nobody waits on a CTA that waits.
//   * Programmatic dependent launch: the producer issues the first stages'
//     weight loads (which no earlier kernel writes) before griddepcontrol.wait,
//     so the previous kernel's tail overlaps this kernel's first HBM reads.
// Epilogues: SwiGLU, residual add (fp32 out), plain fp32, and online-softmax
// statistics per 32-column row block (the [block x token] partials layout the
// finalize kernels read).
#include <atomic>
#include <cfloat>
#include <climits>
#include <cuda.h>
#include "internal.cuh"

namespace ee {

namespace {
constexpr int SD_ROWS = 32;                      // weight rows per row block (= CE block)
constexpr int SD_KC = 256;                       // k per stage: 4 swizzle atoms of 64
constexpr int SD_ATOMS = SD_KC / 64;            // 4 (the atom sums below are written out for 4)
constexpr int SD_W_ATOM = SD_ROWS * 128;         // 4 KB: 32 rows x 128 B
constexpr int SD_CONSUMERS = 4;                  // warps 0-3, 8 weight rows each
constexpr int SD_THREADS = 32 * (SD_CONSUMERS + 1);  // + warp 4: TMA producer
constexpr int SD_MAX_CTAS = 256;
constexpr int SD_SLOTS = 16;                     // launches in flight sharing the fix-up pool

// Stage = NW weight tiles + the [M x 256] activation slice (one 1 KB swizzle
// atom per 64 k for M <= 8 tokens, 2 KB for M <= 16); as many stages as fit in
// ~200 KB of shared memory.  (Measured, profiles/r02x: going from 96 to 200 KB
// in flight did not move a one-tile-per-stage stream off 4.2 TB/s -- two
// far-apart tiles per stage did, see the kernel.)
template <int M, int NW>
struct SdCfg {
  static constexpr int W_BYTES = NW * SD_ATOMS * SD_W_ATOM;
  static constexpr int X_ATOM = (M <= 8 ? 8 : 16) * 128;
  static constexpr int STAGE = W_BYTES + SD_ATOMS * X_ATOM;
  static constexpr int STAGES = (200 * 1024) / STAGE;
  static constexpr int SMEM = 1024 + STAGES * STAGE + 2 * STAGES * 8 + 16 * SD_ROWS * 4;
};

struct SdArgs {
  SkinnyArgs a;
  long long units;  // row blocks x k chunks
  int nkc;          // k chunks per row block
  int nrb;          // row blocks of the matrix
  int half;         // PAIR modes: the second tile of unit row block rb is rb + half
  int slot;         // fix-up pool slot of this launch
  unsigned epoch;   // this launch's flag value in its slot
};

__device__ __forceinline__ uint4 lds128(const uint8_t* p) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(smem_u32(p)));
  return v;
}
__device__ __forceinline__ void consumers_sync() {  // the 4 consumer warps only
  asm volatile("bar.sync 1, %0;" ::"n"(32 * SD_CONSUMERS) : "memory");
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
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

// stream-K fix-up pool: per slot and CTA, the partial accumulators of the row
// block a CTA starts inside of (2 x float4 per consumer thread) and its flag
__device__ float4 g_sd_part[SD_SLOTS][SD_MAX_CTAS][2][SD_CONSUMERS * 32];
__device__ unsigned g_sd_flag[SD_SLOTS][SD_MAX_CTAS];

// out[m][n] = sum_k x[m][k] W[n][k] for m < M <= 16 tokens (SWIGLU: W0 = gate,
// W1 = up; out = silu(x W0^T) * (x W1^T) as bf16).
template <int M, int MODE>
__global__ void __launch_bounds__(SD_THREADS, 1)
    skinny_kernel(const __grid_constant__ CUtensorMap tmW0, const __grid_constant__ CUtensorMap tmW1,
                  const __grid_constant__ CUtensorMap tmX, const SdArgs p) {
  // Every mode streams two weight tiles per stage: SwiGLU the gate and up rows
  // of one row block; the one-matrix modes (PAIR) row blocks rb and rb + half
  // of the same matrix.  Streaming a single 32-row tile (rows 16-56 KB apart)
  // reached only 4.2 TB/s against 6.4-6.5 for two tiles far apart (r02x) --
  // with 200 KB in flight and four MMA chains alike, so the limit is the DRAM
  // side of the access pattern, not the bytes in flight or the consumers.
  constexpr int NW = 2;
  constexpr bool PAIR = MODE != SK_SWIGLU;
  using C = SdCfg<M, NW>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE);
  uint64_t* empty = full + C::STAGES;
  float* s_log = reinterpret_cast<float*>(empty + C::STAGES);  // [16][32] (CE)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long G = gridDim.x, cta = blockIdx.x;
  const long long u0 = p.units * cta / G, u1 = p.units * (cta + 1) / G;
  const int nkc = p.nkc;
  const SkinnyArgs& a = p.a;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], SD_CONSUMERS);
    }
    fence_barrier_init();
  }
  __syncthreads();
  griddep_launch();

  if (warp == SD_CONSUMERS) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      tma_prefetch_desc(&tmW0);
      tma_prefetch_desc(&tmW1);
      tma_prefetch_desc(&tmX);
      constexpr uint32_t tx = C::W_BYTES + SD_ATOMS * M * 128;
      auto load_w = [&](long long u, int s) {
        const int rb = (int)(u / nkc), kc = (int)(u % nkc);
        uint8_t* st = smem + s * C::STAGE;
#pragma unroll
        for (int q = 0; q < SD_ATOMS; ++q) {
          tma_load_2d(st + q * SD_W_ATOM, &tmW0, &full[s], kc * SD_KC + q * 64, rb * SD_ROWS);
          tma_load_2d(st + (SD_ATOMS + q) * SD_W_ATOM, &tmW1, &full[s], kc * SD_KC + q * 64,
                      (rb + p.half) * SD_ROWS);
        }
      };
      auto load_x = [&](long long u, int s) {
        const int kc = (int)(u % nkc);
        uint8_t* st = smem + s * C::STAGE + C::W_BYTES;
#pragma unroll
        for (int q = 0; q < SD_ATOMS; ++q)
          tma_load_2d(st + q * C::X_ATOM, &tmX, &full[s], kc * SD_KC + q * 64, 0);
      };
      const long long n = u1 - u0;
      const int npre = n < C::STAGES ? (int)n : C::STAGES;
      for (int j = 0; j < npre; ++j) {  // weights: written by no earlier kernel
        mbar_arrive_expect_tx(&full[j], tx);
        load_w(u0 + j, j);
      }
      griddep_wait();  // the activations are the previous kernel's output
      for (int j = 0; j < npre; ++j) load_x(u0 + j, j);
      for (long long j = npre; j < n; ++j) {
        const int s = (int)(j % C::STAGES);
        mbar_wait(&empty[s], (uint32_t)((j / C::STAGES - 1) & 1));
        mbar_arrive_expect_tx(&full[s], tx);
        load_w(u0 + j, s);
        load_x(u0 + j, s);
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  griddep_wait();  // resid reads, and output buffers the previous kernel may still read
  const int g = lane >> 2, c = lane & 3;
  const int r = warp * 8 + g;  // weight row within the block (r & 7 == g)
  const uint4 zero = make_uint4(0u, 0u, 0u, 0u);
  const bool tok = g < M, tok1 = M > 8 && g + 8 < M;  // tokens g and g + 8
  long long u = u0, j = 0;
  while (u < u1) {
    const int rb = (int)(u / nkc);
    const long long rb_end = (long long)(rb + 1) * nkc;
    const long long stop = rb_end < u1 ? rb_end : u1;
    // one accumulator per 64-k atom: four independent MMA chains per warp (a
    // single chain made the 4 consumer warps MMA-latency-bound, ~1100 cycles
    // per 16 KB stage: 4.2 TB/s for the one-matrix modes; r02x)
    float e0[SD_ATOMS][4], e1[SD_ATOMS][4];
#pragma unroll
    for (int q = 0; q < SD_ATOMS; ++q)
#pragma unroll
      for (int v = 0; v < 4; ++v) e0[q][v] = e1[q][v] = 0.f;
    for (; u < stop; ++u, ++j) {
      const int s = (int)(j % C::STAGES);
      mbar_wait(&full[s], (uint32_t)((j / C::STAGES) & 1));
      const uint8_t* st = smem + s * C::STAGE;
      const uint8_t* sx = st + C::W_BYTES;
#pragma unroll
      for (int q = 0; q < SD_ATOMS; ++q) {
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int sw = ((hh * 4 + c) ^ g) << 4;  // 128B swizzle: chunk ^ (row & 7)
          const uint4 w = lds128(st + q * SD_W_ATOM + r * 128 + sw);
          const uint4 x0 = tok ? lds128(sx + q * C::X_ATOM + g * 128 + sw) : zero;
          const uint4 x1 = tok1 ? lds128(sx + q * C::X_ATOM + (g + 8) * 128 + sw) : zero;
          mma_chunk(e0[q], x0, x1, w);
          const uint4 w1 = lds128(st + (SD_ATOMS + q) * SD_W_ATOM + r * 128 + sw);
          mma_chunk(e1[q], x0, x1, w1);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    float d0[4], d1[4];  // fixed-order sum over the atoms' accumulators
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      d0[v] = ((e0[0][v] + e0[1][v]) + e0[2][v]) + e0[3][v];
      d1[v] = ((e1[0][v] + e1[1][v]) + e1[2][v]) + e1[3][v];
    }
    const int tid = warp * 32 + lane;
    if ((long long)rb * nkc < u0) {
      // this CTA started inside row block rb: publish the partial sums for the
      // CTA that holds rb's first chunk (happens once, at the start of the range)
      g_sd_part[p.slot][cta][0][tid] = make_float4(d0[0], d0[1], d0[2], d0[3]);
      g_sd_part[p.slot][cta][1][tid] = make_float4(d1[0], d1[1], d1[2], d1[3]);
      __threadfence();
      consumers_sync();
      if (tid == 0) st_release_u32(&g_sd_flag[p.slot][cta], p.epoch);
      continue;
    }
    // finisher: add the contributions of the later CTAs starting inside rb, in CTA order
    for (long long q = cta + 1; q < G; ++q) {
      if (p.units * q / G >= rb_end) break;
      // bounded wait: the contributor is resident or about to be (one CTA per
      // SM, grid <= SMs); only co-running kernels that never yield could hold
      // it off, and then the call fails (status) instead of hanging
      if (ld_acquire_u32(&g_sd_flag[p.slot][q]) != p.epoch) {
        const unsigned long long t0 = globaltimer_ns();
        while (ld_acquire_u32(&g_sd_flag[p.slot][q]) != p.epoch) {
          __nanosleep(32);
          if (globaltimer_ns() - t0 > 5000000000ull) {
            if (p.a.st && tid == 0) set_status(p.a.st, 9 /* EE_ERR_CUDA */, -1);
            break;
          }
        }
      }
      const float4 v = __ldcg(&g_sd_part[p.slot][q][0][tid]);
      d0[0] += v.x; d0[1] += v.y; d0[2] += v.z; d0[3] += v.w;
      const float4 w = __ldcg(&g_sd_part[p.slot][q][1][tid]);
      d1[0] += w.x; d1[1] += w.y; d1[2] += w.z; d1[3] += w.w;
    }
    // d[0], d[1] = out[token g][n0 + 2c (+1)]; d[2], d[3] = out[token g + 8][...]
    auto epilogue = [&](int rbx, const float (&v0)[4], const float (&v1)[4]) {
      const int na = rbx * SD_ROWS + warp * 8 + 2 * c;
      if constexpr (MODE == SK_CE) {
        if (tok) {
          s_log[g * SD_ROWS + warp * 8 + 2 * c] = na < a.N ? v0[0] : -INFINITY;
          s_log[g * SD_ROWS + warp * 8 + 2 * c + 1] = na + 1 < a.N ? v0[1] : -INFINITY;
        }
        if (tok1) {
          s_log[(g + 8) * SD_ROWS + warp * 8 + 2 * c] = na < a.N ? v0[2] : -INFINITY;
          s_log[(g + 8) * SD_ROWS + warp * 8 + 2 * c + 1] = na + 1 < a.N ? v0[3] : -INFINITY;
        }
        consumers_sync();
        for (int m = warp; m < M; m += SD_CONSUMERS) {  // token m's statistics over 32 columns
          const float v = s_log[m * SD_ROWS + lane];
          float mx = v;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
          float se = v == -INFINITY ? 0.f : __expf(v - mx);
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
          const unsigned ball = __ballot_sync(0xffffffffu, v == mx);
          if (lane == 0) {
            a.pm[(long long)rbx * M + m] = mx;
            a.ps[(long long)rbx * M + m] = se;
            a.pi[(long long)rbx * M + m] = a.vocab_begin + rbx * SD_ROWS + (__ffs(ball) - 1);
          }
        }
        consumers_sync();  // s_log is rewritten by the next row block
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int tk = g + (e >= 2 ? 8 : 0);
          const int n = na + (e & 1);
          if (!(e >= 2 ? tok1 : tok) || n >= a.N) continue;
          const long long o = (long long)tk * a.ldo + n;
          if constexpr (MODE == SK_SWIGLU) {
            const float v = v0[e], w = v1[e];
            a.outb[o] = __float2bfloat16_rn(__fdividef(v, 1.0f + __expf(-v)) * w);
          } else if constexpr (MODE == SK_RESID) {
            a.out[o] = v0[e] + __bfloat162float(a.resid[(long long)tk * a.ldr + n]);
          } else {
            a.out[o] = v0[e];
          }
        }
      }
    };
    if constexpr (PAIR) {  // two row blocks: rb and rb + half (if it exists)
      epilogue(rb, d0, d0);
      if (rb + p.half < p.nrb) epilogue(rb + p.half, d1, d1);
    } else {
      epilogue(rb, d0, d1);
    }
  }
}

namespace {
std::atomic<unsigned> g_sd_launches{0};

template <int M, int MODE>
cudaError_t launch_mm(const CUtensorMap& w0, const CUtensorMap& w1, const CUtensorMap& x,
                      const SdArgs& p, int grid, cudaStream_t s) {
  constexpr int NW = 2;
  auto kern = skinny_kernel<M, MODE>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         SdCfg<M, NW>::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  return launch_pdl(kern, dim3(grid), dim3(SD_THREADS), SdCfg<M, NW>::SMEM, s, w0, w1, x, p);
}

template <int MODE>
cudaError_t launch_m(const SkinnyArgs& a, int M, cudaStream_t s) {
  CUtensorMap tw0, tw1, tx;
  if (!make_tmap(&tw0, Mat{a.W0, a.N, a.K, a.K}, 64, SD_ROWS)) return cudaErrorInvalidValue;
  if (MODE == SK_SWIGLU) {
    if (!make_tmap(&tw1, Mat{a.W1, a.N, a.K, a.K}, 64, SD_ROWS)) return cudaErrorInvalidValue;
  } else {
    tw1 = tw0;
  }
  if (!make_tmap(&tx, Mat{a.x, M, a.K, a.ldx}, 64, (uint32_t)M)) return cudaErrorInvalidValue;
  SdArgs p{};
  p.a = a;
  p.nkc = (a.K + SD_KC - 1) / SD_KC;
  p.nrb = (a.N + SD_ROWS - 1) / SD_ROWS;
  p.half = MODE == SK_SWIGLU ? 0 : (p.nrb + 1) / 2;
  p.units = (long long)(MODE == SK_SWIGLU ? p.nrb : p.half) * p.nkc;
  long long grid = num_sms();
  if (grid > SD_MAX_CTAS) grid = SD_MAX_CTAS;
  if (grid > p.units) grid = p.units;
  const unsigned id = g_sd_launches.fetch_add(1);
  p.slot = (int)(id % SD_SLOTS);
  p.epoch = id / SD_SLOTS + 1;
  switch (M) {
#define EE_SK(m) case m: return launch_mm<m, MODE>(tw0, tw1, tx, p, (int)grid, s);
    EE_SK(1) EE_SK(2) EE_SK(3) EE_SK(4) EE_SK(5) EE_SK(6) EE_SK(7) EE_SK(8)
    EE_SK(9) EE_SK(10) EE_SK(11) EE_SK(12) EE_SK(13) EE_SK(14) EE_SK(15) EE_SK(16)
#undef EE_SK
  }
  return cudaErrorInvalidValue;
}
}  // namespace

int skinny_blocks(int N) { return (N + SD_ROWS - 1) / SD_ROWS; }

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
  griddep_launch();
  griddep_wait();
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
  return launch_pdl(infer_finalize_wide_kernel, dim3(M), dim3(256), 0, s, pm, ps, pi, nb, M, lse,
                    argmax, conf);
}

cudaError_t launch_skinny(int mode, const SkinnyArgs& a, int M, cudaStream_t s) {
  if (M < 1 || M > SKINNY_MAX_M || a.K % 8 != 0 || a.ldx % 8 != 0) return cudaErrorInvalidValue;
  switch (mode) {
    case SK_F32: return launch_m<SK_F32>(a, M, s);
    case SK_RESID: return launch_m<SK_RESID>(a, M, s);
    case SK_SWIGLU: return launch_m<SK_SWIGLU>(a, M, s);
    case SK_CE: return launch_m<SK_CE>(a, M, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace ee
