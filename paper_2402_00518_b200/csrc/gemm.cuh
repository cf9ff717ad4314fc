// gemm.cuh -- persistent, warp-specialised tcgen05 GEMM for sm_100a with the
// fused epilogues of the EE-Tuning exit-head step.
//
//   D[M x N] = A[M x K] * B[N x K]^T        (bf16 operands, fp32 accumulate in TMEM)
//
// A and B are each either K-major (K contiguous) or MN-major (M/N contiguous)
// in global memory, so every GEMM of the step -- forward (z W_out^T), input
// gradients (dS W_out) and weight gradients (dS^T z) -- reads its operands in
// place with no transposes (UMMA descriptor "major" bits).
//
// Tile 128 x 256 x 64, 4-stage TMA->SMEM ring (128B swizzle), accumulator
// double-buffered in TMEM (2 x 256 columns), one CTA per SM, static persistent
// tile schedule with grouped rasterisation.  Warp roles (256 threads):
//   warp 0     TMA producer (lane 0)
//   warp 1     MMA issuer   (lane 0): 4 x tcgen05.mma (K=16) per stage
//   warp 2     TMEM allocator
//   warps 4-7  epilogue: thread t <-> TMEM lane t <-> one output row; the
//              whole 256-column row slice of a tile is thread-local, which is
//              what makes the online-softmax statistics shuffle-free.
#pragma once
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include "ptx.cuh"

namespace ee {

constexpr int GEMM_BM = 128;
constexpr int GEMM_BN = 256;
constexpr int GEMM_BK = 64;
constexpr int GEMM_STAGES = 4;
constexpr int GEMM_THREADS = 256;
constexpr int GEMM_A_STAGE = GEMM_BM * GEMM_BK * 2;  // 16 KB
constexpr int GEMM_B_STAGE = GEMM_BN * GEMM_BK * 2;  // 32 KB
constexpr int GEMM_SMEM = GEMM_STAGES * (GEMM_A_STAGE + GEMM_B_STAGE) + 1024 + 256;
constexpr int GEMM_TMEM_COLS = 512;

enum EpiKind : int {
  EPI_F32 = 0,         // out = acc (or out += acc), fp32, rows split over two pointers
  EPI_RESID = 1,       // out = resid(bf16) + acc, fp32           (MLP down proj, residual)
  EPI_SWIGLU_FWD = 2,  // [gate|up] tile -> A, B (bf16) and M = silu(A)*B (bf16)
  EPI_SWIGLU_BWD = 3,  // acc = dM; dA = dM*B*silu'(A), dB = dM*silu(A) in place over A, B
  EPI_CE_STATS = 4,    // per-row (max, sum exp, argmax) of the tile + target logit
  EPI_CE_DS = 5,       // dS = coef * (exp(S - lse) - onehot(y)) -> bf16
  EPI_F32T = 6,        // out^T: out[n][m] = acc (or +=), columns n >= n_split go to out1
  EPI_BF16 = 7,        // outb[m][n] = bf16(acc)   (backbone projections)
  EPI_F32_ADAM = 8,    // EPI_F32 whose finished tile is a gradient: Adam in place (adam0/1)
  EPI_F32T_ADAM = 9,   // EPI_F32T likewise (ee_tune_step_adam)
};

enum BMode : int {
  B_PLAIN = 0,   // B tile = 256 rows of tmB0
  B_PAIR = 1,    // B tile rows [0,128) from tmB0, [128,256) from tmB1, same n offset (gate|up)
  B_KSPLIT = 2,  // k < b_ksplit from tmB0, k >= b_ksplit from tmB1 (K concatenation)
};

// Adam (A14) on one element, with explicit roundings so
// the standalone adam_kernel and the fused weight-gradient epilogue
// (ee_tune_step_adam) produce the same bits.
struct AdamScal {
  float lr, b1, b2, eps, wd, bc1, bc2, gs;
};
__device__ __forceinline__ void adam_update(float& th, float& m, float& v, float g,
                                            const AdamScal& s) {
  g = __fmul_rn(s.gs, g);
  m = __fmaf_rn(s.b1, m, __fmul_rn(__fsub_rn(1.f, s.b1), g));
  v = __fmaf_rn(s.b2, v, __fmul_rn(__fmul_rn(__fsub_rn(1.f, s.b2), g), g));
  const float upd = __fdiv_rn(__fdiv_rn(m, s.bc1), __fadd_rn(__fsqrt_rn(__fdiv_rn(v, s.bc2)), s.eps));
  th = __fsub_rn(__fsub_rn(th, __fmul_rn(s.lr, upd)), __fmul_rn(__fmul_rn(s.lr, s.wd), th));
}
// Parameter state one output of a fused-Adam GEMM updates (row-major like the
// gradient it replaces): fp32 master, moments, bf16 operand copy.
struct AdamOut {
  float *th, *m, *v;
  __nv_bfloat16* op;
};

struct GemmArgs {
  int M, N, K;  // N = logical output columns (B_PAIR: columns of each of the two halves)
  int m_blocks, n_blocks, k_blocks;
  int b_mode, b_ksplit, group_m;
  int hint_a, hint_b;
  int epi_sleep;  // epilogue accumulator wait: 0 spin, 1 try_wait suspend hint, >= 2 poll + nanosleep(epi_sleep ns)
  int* tile_counter;  // CTA-pair kernel: dynamic tile schedule counter (zeroed per launch), or NULL
  int* wave_counter;  // CTA-pair kernel, static schedule: per-wave soft barrier counter, or NULL
  unsigned long long* trace;  // debug: per-tile (globaltimer << 8 | smid) at accumulator-ready, or NULL  // L2 policy of the A / B TMA loads: -1 none, 0 normal, 1 evict_last, 2 evict_first
  // EPI_F32 / EPI_RESID
  float* out0;
  float* out1;
  long long ldo;
  int m_split;
  int n_split;  // EPI_F32T: output columns n >= n_split go to out1 (row n - n_split)
  int accumulate;
  // Fused reduce-scatter (scat_rows > 0; out0/out1 unused): stored row r of
  // the output goes to the owner q = r / scat_rows of that row block, at
  // scat[q] + (r - q * scat_rows) * ldo (scat1 for EPI_F32T rows >= n_split).
  // The host folds this rank's slot offset into each pointer (include/ee.h
  // ee_vp_vocab_backward_rs: dz rows to token owners; ee_tune_step_rs:
  // gradient rows to parameter-shard owners).  EPI_F32: stored row = m;
  // EPI_F32T: stored row = n.
  float* scat[8];
  float* scat1[8];
  int scat_rows;
  // Fused Adam (adam_on; EPI_F32 / EPI_F32T, accumulate = 0): the finished
  // accumulator tile IS the gradient; instead of storing it, update
  // adam0 (rows < m_split / columns < n_split) or adam1 in place.
  int adam_on;
  AdamScal adam;
  AdamOut adam0, adam1;
  // EPI_F32T / EPI_F32T_ADAM gain identity (MLP exits; DESIGN.md §3 A28):
  // when row_scale != NULL every accumulator row m is
  // multiplied by row_scale[m] before it is stored or updated (dW_gate|up =
  // g_a (.) ([dA|dB]^T x^) when the A operand is x^ = x r), and, when
  // gain_part != NULL, gain_part[nb * M + m] receives sum over the tile's
  // columns n of gw(n)[n'][m] * acc[m][n] (unscaled; gw = gain_w0 for
  // n < n_split, n' = n, else gain_w1, n' = n - n_split; bf16 [rows x M]):
  // the pre-MLP gain's gradient sum_t du_t (.) x^_t without forming du.
  const float* row_scale;
  float* gain_part;
  const __nv_bfloat16* gain_w0;
  const __nv_bfloat16* gain_w1;
  const __nv_bfloat16* resid;
  long long ld_resid;
  __nv_bfloat16* outb;  // EPI_BF16 output (ldo)
  int rope_seq;         // EPI_BF16: > 0 = apply RoPE (rotate-half, head dim 128; N % 128 == 0)
  float rope_theta;     //   at position row % rope_seq before the bf16 rounding
  const float2* rope_tab;  // (cos, sin) [rope_seq x 64] (launch_rope_table); NULL: computed
  // SwiGLU
  __nv_bfloat16* ab;  // [M x 2F]: A in columns [0,F), B in [F,2F)
  long long ld_ab;
  __nv_bfloat16* mact;  // [M x F]
  long long ld_m;
  int ffn;
  // cross-entropy
  const int32_t* targets;
  int vocab_begin;
  float* part_m;
  float* part_s;
  int32_t* part_i;
  float* tgt_logit;
  const float* lse;
  const float* coef;
  __nv_bfloat16* ds;
  long long ld_ds;
};

__device__ __forceinline__ void tile_coords(const GemmArgs& a, int tile, int& mb, int& nb) {
  const int group_size = a.group_m * a.n_blocks;
  const int g = tile / group_size;
  const int first_m = g * a.group_m;
  const int gm = min(a.m_blocks - first_m, a.group_m);
  const int r = tile - g * group_size;
  mb = first_m + r % gm;
  nb = r / gm;
}

__device__ __forceinline__ float u2f(uint32_t v) { return __uint_as_float(v); }

__device__ __forceinline__ unsigned long long trace_stamp() {
  unsigned long long t;
  uint32_t sm;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
  return (t << 8) | (sm & 0xFF);
}

// 16 bf16 (32 bytes): one 256-bit store when aligned, else two 128-bit stores.
__device__ __forceinline__ void store16_bf16(__nv_bfloat16* p, const uint32_t (&w)[8]) {
  if (aligned32(p)) {
    st_global_v8(p, w);
  } else {
    *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
    *reinterpret_cast<uint4*>(p + 8) = make_uint4(w[4], w[5], w[6], w[7]);
  }
}

// Epilogue of one accumulator tile: thread `row` of the 128 epilogue threads
// owns TMEM lane `row` = output row gm; `tb` = TMEM address of this warp's
// lane quarter in the accumulator stage; nb = N-block of the tile.
template <int EPI>
__device__ __forceinline__ void epilogue_tile(const GemmArgs& args, uint32_t tb, int gm, int nb) {
  const bool row_ok = gm < args.M;
  if constexpr (EPI == EPI_F32 || EPI == EPI_RESID || EPI == EPI_F32_ADAM) {
    float* orow = nullptr;
    if (row_ok) {
      if (EPI != EPI_RESID && args.scat_rows > 0) {
        const int q = gm / args.scat_rows;
        orow = args.scat[q] + (long long)(gm - q * args.scat_rows) * args.ldo;
      } else {
        orow = (gm < args.m_split) ? args.out0 + (long long)gm * args.ldo
                                   : args.out1 + (long long)(gm - args.m_split) * args.ldo;
      }
    }
#pragma unroll 1
    for (int c = 0; c < GEMM_BN / 32; ++c) {
      uint32_t v[32];
      tmem_ld_32x32b_x32(tb + c * 32, v);
      tmem_ld_wait();
      const int gn0 = nb * GEMM_BN + c * 32;
      if (row_ok && gn0 < args.N) {
#pragma unroll
        for (int j = 0; j < 32; j += 8) {
          const int gn = gn0 + j;
          if (gn >= args.N) continue;
          float o[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) o[q] = u2f(v[j + q]);
          const bool full8 = gn + 8 <= args.N;
          if constexpr (EPI == EPI_RESID) {
            const __nv_bfloat16* rp = args.resid + (long long)gm * args.ld_resid + gn;
            const uint2 r0 = *reinterpret_cast<const uint2*>(rp);
            o[0] += bf16lo(r0.x); o[1] += bf16hi(r0.x); o[2] += bf16lo(r0.y); o[3] += bf16hi(r0.y);
            if (full8) {
              const uint2 r1 = *reinterpret_cast<const uint2*>(rp + 4);
              o[4] += bf16lo(r1.x); o[5] += bf16hi(r1.x); o[6] += bf16lo(r1.y); o[7] += bf16hi(r1.y);
            }
          } else {
            if (args.accumulate) {
              const float4 p0 = *reinterpret_cast<const float4*>(orow + gn);
              o[0] += p0.x; o[1] += p0.y; o[2] += p0.z; o[3] += p0.w;
              if (full8) {
                const float4 p1 = *reinterpret_cast<const float4*>(orow + gn + 4);
                o[4] += p1.x; o[5] += p1.y; o[6] += p1.z; o[7] += p1.w;
              }
            }
          }
          if constexpr (EPI == EPI_F32_ADAM) {  // fused Adam on the finished gradient
            const bool lo = gm < args.m_split;
            const AdamOut& ao = lo ? args.adam0 : args.adam1;
            const long long e = (long long)(lo ? gm : gm - args.m_split) * args.ldo + gn;
            // 8 consecutive elements (e % 8 == 0: ldo and gn are multiples of 8):
            // 16-byte loads of all three states first, then the update and stores
            float th[8], mm[8], vv[8];
            const int nq = full8 ? 2 : 1;
#pragma unroll
            for (int h4 = 0; h4 < 2; ++h4)
              if (h4 < nq) {
                const float4 a = *reinterpret_cast<const float4*>(ao.th + e + 4 * h4);
                const float4 b = *reinterpret_cast<const float4*>(ao.m + e + 4 * h4);
                const float4 c = *reinterpret_cast<const float4*>(ao.v + e + 4 * h4);
                th[4 * h4] = a.x; th[4 * h4 + 1] = a.y; th[4 * h4 + 2] = a.z; th[4 * h4 + 3] = a.w;
                mm[4 * h4] = b.x; mm[4 * h4 + 1] = b.y; mm[4 * h4 + 2] = b.z; mm[4 * h4 + 3] = b.w;
                vv[4 * h4] = c.x; vv[4 * h4 + 1] = c.y; vv[4 * h4 + 2] = c.z; vv[4 * h4 + 3] = c.w;
              }
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if (q < 4 * nq) adam_update(th[q], mm[q], vv[q], o[q], args.adam);
#pragma unroll
            for (int h4 = 0; h4 < 2; ++h4)
              if (h4 < nq) {
                *reinterpret_cast<float4*>(ao.th + e + 4 * h4) =
                    make_float4(th[4 * h4], th[4 * h4 + 1], th[4 * h4 + 2], th[4 * h4 + 3]);
                *reinterpret_cast<float4*>(ao.m + e + 4 * h4) =
                    make_float4(mm[4 * h4], mm[4 * h4 + 1], mm[4 * h4 + 2], mm[4 * h4 + 3]);
                *reinterpret_cast<float4*>(ao.v + e + 4 * h4) =
                    make_float4(vv[4 * h4], vv[4 * h4 + 1], vv[4 * h4 + 2], vv[4 * h4 + 3]);
                *reinterpret_cast<uint2*>(ao.op + e + 4 * h4) =
                    make_uint2(pack_bf16(th[4 * h4], th[4 * h4 + 1]),
                               pack_bf16(th[4 * h4 + 2], th[4 * h4 + 3]));
              }
            continue;
          } else {
          if (full8 && aligned32(orow + gn)) {
            uint32_t w[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) w[q] = __float_as_uint(o[q]);
            st_global_v8(orow + gn, w);
          } else {
            *reinterpret_cast<float4*>(orow + gn) = make_float4(o[0], o[1], o[2], o[3]);
            if (full8) *reinterpret_cast<float4*>(orow + gn + 4) = make_float4(o[4], o[5], o[6], o[7]);
          }
          }
        }
      }
    }
  } else if constexpr (EPI == EPI_BF16) {
    __nv_bfloat16* orow = row_ok ? args.outb + (long long)gm * args.ldo : nullptr;
    if (args.rope_seq > 0) {
      // Fused RoPE (Llama rotate-half): the N-tile holds GEMM_BN / 128 whole
      // heads, and this thread holds both x_i and x_{i+64} of each for its row;
      // rotate in fp32 by angle pos * theta^(-2i/128), then round to bf16 once.
      const float pos = (float)(gm % args.rope_seq);
#pragma unroll 1
      for (int hc = 0; hc < (GEMM_BN / 128) * 2; ++hc) {
        const int hd = hc >> 1, c = hc & 1;  // head within the tile, 32-column chunk
        if (nb * GEMM_BN + hd * 128 >= args.N) break;
        // one load per wait: the asm outputs are only valid after wait::ld
        uint32_t v0[32], v1[32];
        tmem_ld_32x32b_x32(tb + hd * 128 + c * 32, v0);
        tmem_ld_wait();
        tmem_ld_32x32b_x32(tb + hd * 128 + (c + 2) * 32, v1);
        tmem_ld_wait();
        if (!row_ok) continue;
        uint32_t w0[2][8], w1[2][8];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          float ra[2], rb[2];
#pragma unroll
          float csn[4];  // cos_i, sin_i, cos_i+1, sin_i+1
          if (args.rope_tab) {
            const float4 t4 = *reinterpret_cast<const float4*>(
                args.rope_tab + (long long)(gm % args.rope_seq) * 64 + c * 32 + 2 * q);
            csn[0] = t4.x; csn[1] = t4.y; csn[2] = t4.z; csn[3] = t4.w;
          } else {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const float inv = powf(args.rope_theta, -2.0f * (float)(c * 32 + 2 * q + e) / 128.0f);
              sincosf(pos * inv, &csn[2 * e + 1], &csn[2 * e]);
            }
          }
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const float cs = csn[2 * e], sn = csn[2 * e + 1];
            const float a = u2f(v0[2 * q + e]), b = u2f(v1[2 * q + e]);
            ra[e] = a * cs - b * sn;
            rb[e] = b * cs + a * sn;
          }
          w0[q >> 3][q & 7] = pack_bf16(ra[0], ra[1]);
          w1[q >> 3][q & 7] = pack_bf16(rb[0], rb[1]);
        }
        __nv_bfloat16* p0 = orow + nb * GEMM_BN + hd * 128 + c * 32;
        store16_bf16(p0, w0[0]);
        store16_bf16(p0 + 16, w0[1]);
        store16_bf16(p0 + 64, w1[0]);
        store16_bf16(p0 + 80, w1[1]);
      }
      return;
    }
#pragma unroll 1
    for (int c = 0; c < GEMM_BN / 32; ++c) {
      uint32_t v[32];
      tmem_ld_32x32b_x32(tb + c * 32, v);
      tmem_ld_wait();
      const int gn0 = nb * GEMM_BN + c * 32;
      if (row_ok && gn0 < args.N) {
#pragma unroll
        for (int j = 0; j < 32; j += 16) {
          if (gn0 + j >= args.N) continue;
          uint32_t w[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) w[q] = pack_bf16(u2f(v[j + 2 * q]), u2f(v[j + 2 * q + 1]));
          __nv_bfloat16* p = orow + gn0 + j;
          if (gn0 + j + 16 <= args.N && aligned32(p)) {
            st_global_v8(p, w);
          } else {
            *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
            if (gn0 + j + 8 < args.N)
              *reinterpret_cast<uint4*>(p + 8) = make_uint4(w[4], w[5], w[6], w[7]);
          }
        }
      }
    }
  } else if constexpr (EPI == EPI_F32T || EPI == EPI_F32T_ADAM) {
    // Transposed store: the tile is D' = A'B'^T computed with the operands
    // swapped so that A' is K-major (the fast UMMA path); the caller's output
    // is D'^T.  Thread `row` (m) writes out[n][m]: for each n the 32 threads of
    // a warp store 32 consecutive floats (one 128-byte line).
    float gsum = 0.f;   // gain identity: this row's sum over the tile's columns
#pragma unroll 1
    for (int c = 0; c < GEMM_BN / 32; ++c) {
      uint32_t v[32];
      tmem_ld_32x32b_x32(tb + c * 32, v);
      tmem_ld_wait();
      const int gn0 = nb * GEMM_BN + c * 32;
      if (args.row_scale != nullptr && row_ok) {
        // gw[n'][m] over the 32 threads of a warp (consecutive m) is one
        // coalesced 64-byte segment per n
        const float rs = args.row_scale[gm];
        if (args.gain_part != nullptr) {
          // the 32 weight values first (read-only loads, all in flight at once),
          // then the fixed-order FMA chain: issued one by one behind the FMAs
          // they exposed a full L2 latency each, and at K = 8192 (DP over 8
          // ranks) the epilogue outlasted the mainloop (ncu, profiles/r02dp8)
          // (asm volatile keeps the 32 loads in issue order ahead of their first
          // use -- with plain loads nvcc reused one register and waited on
          // each; indices past N are clamped, their products skipped)
          uint16_t wraw[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int gn = min(gn0 + j, args.N - 1);
            const __nv_bfloat16* w = gn < args.n_split
                                         ? args.gain_w0 + (long long)gn * args.M + gm
                                         : args.gain_w1 + (long long)(gn - args.n_split) * args.M + gm;
            asm volatile("ld.global.nc.u16 %0, [%1];" : "=h"(wraw[j]) : "l"(w));
          }
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (gn0 + j < args.N)
              gsum = fmaf(__uint_as_float(static_cast<uint32_t>(wraw[j]) << 16), u2f(v[j]), gsum);
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(u2f(v[j]) * rs);
      }
      if (EPI == EPI_F32T_ADAM && row_ok && gn0 < args.N) {
        // fused Adam, element (row n, column m): 16 columns per batch, all 48
        // state loads issued before the updates and stores (each is a
        // 128-byte warp-coalesced row segment); batches never straddle n_split
        // (host: n_split % 16 == 0)
#pragma unroll
        for (int jb = 0; jb < 32; jb += 16) {
          const int gb = gn0 + jb;
          if (gb >= args.N) continue;
          const bool lo = gb < args.n_split;
          const AdamOut& ao = lo ? args.adam0 : args.adam1;
          const long long e0 = (long long)(lo ? gb : gb - args.n_split) * args.ldo + gm;
          float th[16], mm[16], vv[16];
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (gb + j < args.N) {
              const long long e = e0 + (long long)j * args.ldo;
              th[j] = ao.th[e]; mm[j] = ao.m[e]; vv[j] = ao.v[e];
            }
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (gb + j < args.N) {
              adam_update(th[j], mm[j], vv[j], u2f(v[jb + j]), args.adam);
              const long long e = e0 + (long long)j * args.ldo;
              ao.th[e] = th[j]; ao.m[e] = mm[j]; ao.v[e] = vv[j];
              ao.op[e] = __float2bfloat16_rn(th[j]);
            }
        }
      } else if (row_ok && gn0 < args.N) {
        bool done = false;
        if (args.scat_rows > 0) {
          // the usual case: the 32 stored rows of this chunk lie in one owner's
          // block on one side of n_split -> one base pointer, no per-element division
          const int last = min(gn0 + 31, args.N - 1);
          const bool hi0 = gn0 >= args.n_split, hi1 = last >= args.n_split;
          const int r0 = hi0 ? gn0 - args.n_split : gn0;
          const int r1 = hi1 ? last - args.n_split : last;
          const int q0 = r0 / args.scat_rows;
          if (hi0 == hi1 && q0 == r1 / args.scat_rows) {
            float* base = (hi0 ? args.scat1[q0] : args.scat[q0]) +
                          (long long)(r0 - q0 * args.scat_rows) * args.ldo + gm;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              if (gn0 + j < args.N) {
                float* o = base + (long long)j * args.ldo;
                const float val = u2f(v[j]);
                *o = args.accumulate ? *o + val : val;
              }
            }
            done = true;
          }
        }
#pragma unroll
        for (int j = 0; j < 32 && !done; ++j) {
          const int gn = gn0 + j;
          if (gn < args.N) {
            float* o;
            if (args.scat_rows > 0) {  // fused reduce-scatter to the row-block owner
              const bool hi = gn >= args.n_split;
              const int r = hi ? gn - args.n_split : gn;
              const int q = r / args.scat_rows;
              o = (hi ? args.scat1[q] : args.scat[q]) + (long long)(r - q * args.scat_rows) * args.ldo + gm;
            } else {
              o = (gn < args.n_split) ? args.out0 + (long long)gn * args.ldo + gm
                                      : args.out1 + (long long)(gn - args.n_split) * args.ldo + gm;
            }
            const float val = u2f(v[j]);
            *o = args.accumulate ? *o + val : val;
          }
        }
      }
    }
    if (args.gain_part != nullptr && row_ok) args.gain_part[(long long)nb * args.M + gm] = gsum;
  } else if constexpr (EPI == EPI_SWIGLU_FWD) {
    const int F = args.ffn;
#pragma unroll 1
    for (int c = 0; c < GEMM_BN / 64; ++c) {
      uint32_t g[32], u[32];
      tmem_ld_32x32b_x32(tb + c * 32, g);
      tmem_ld_32x32b_x32(tb + GEMM_BN / 2 + c * 32, u);
      tmem_ld_wait();
      const int f0 = nb * (GEMM_BN / 2) + c * 32;
      if (row_ok && f0 < args.N) {
        __nv_bfloat16* arow = args.ab + (long long)gm * args.ld_ab;
        __nv_bfloat16* mrow = args.mact + (long long)gm * args.ld_m;
#pragma unroll
        for (int j = 0; j < 32; j += 16) {
          uint32_t qa[8], qb[8], qm[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float a0 = u2f(g[j + 2 * q]), a1 = u2f(g[j + 2 * q + 1]);
            const float b0 = u2f(u[j + 2 * q]), b1 = u2f(u[j + 2 * q + 1]);
            // fast division (MUFU.RCP + FMUL): the IEEE one's Newton steps and
            // slow-path branch made the SwiGLU epilogues outlast short-K mainloops
            const float s0 = __fdividef(a0, 1.0f + __expf(-a0));
            const float s1 = __fdividef(a1, 1.0f + __expf(-a1));
            qa[q] = pack_bf16(a0, a1);
            qb[q] = pack_bf16(b0, b1);
            qm[q] = pack_bf16(s0 * b0, s1 * b1);
          }
          __nv_bfloat16* pa = arow + f0 + j;
          __nv_bfloat16* pb = arow + F + f0 + j;
          __nv_bfloat16* pm = mrow + f0 + j;
          if (aligned32(pa) && aligned32(pb) && aligned32(pm)) {
            st_global_v8(pa, qa);
            st_global_v8(pb, qb);
            st_global_v8(pm, qm);
          } else {
            *reinterpret_cast<uint4*>(pa) = make_uint4(qa[0], qa[1], qa[2], qa[3]);
            *reinterpret_cast<uint4*>(pa + 8) = make_uint4(qa[4], qa[5], qa[6], qa[7]);
            *reinterpret_cast<uint4*>(pb) = make_uint4(qb[0], qb[1], qb[2], qb[3]);
            *reinterpret_cast<uint4*>(pb + 8) = make_uint4(qb[4], qb[5], qb[6], qb[7]);
            *reinterpret_cast<uint4*>(pm) = make_uint4(qm[0], qm[1], qm[2], qm[3]);
            *reinterpret_cast<uint4*>(pm + 8) = make_uint4(qm[4], qm[5], qm[6], qm[7]);
          }
        }
      }
    }
  } else if constexpr (EPI == EPI_SWIGLU_BWD) {
    const int F = args.ffn;
#pragma unroll 1
    for (int c = 0; c < GEMM_BN / 32; ++c) {
      uint32_t v[32];
      tmem_ld_32x32b_x32(tb + c * 32, v);
      tmem_ld_wait();
      const int f0 = nb * GEMM_BN + c * 32;
      if (row_ok && f0 < args.N) {
        __nv_bfloat16* arow = args.ab + (long long)gm * args.ld_ab;
        // both 16-column halves' A / B loads first, then the math, then the
        // stores: the in-place stores (asm volatile, "memory") otherwise kept
        // the second half's loads behind the first half's stores -- one memory
        // latency per 16 columns
        uint32_t qa[2][8], qb[2][8];
        bool v8[2];
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          __nv_bfloat16* pa_ = arow + f0 + 16 * hf;
          __nv_bfloat16* pb_ = arow + F + f0 + 16 * hf;
          v8[hf] = aligned32(pa_) && aligned32(pb_);
          if (v8[hf]) {
            ld_global_v8(pa_, qa[hf]);
            ld_global_v8(pb_, qb[hf]);
          } else {
            const uint4 a0 = *reinterpret_cast<const uint4*>(pa_);
            const uint4 a1 = *reinterpret_cast<const uint4*>(pa_ + 8);
            const uint4 b0 = *reinterpret_cast<const uint4*>(pb_);
            const uint4 b1 = *reinterpret_cast<const uint4*>(pb_ + 8);
            qa[hf][0] = a0.x; qa[hf][1] = a0.y; qa[hf][2] = a0.z; qa[hf][3] = a0.w;
            qa[hf][4] = a1.x; qa[hf][5] = a1.y; qa[hf][6] = a1.z; qa[hf][7] = a1.w;
            qb[hf][0] = b0.x; qb[hf][1] = b0.y; qb[hf][2] = b0.z; qb[hf][3] = b0.w;
            qb[hf][4] = b1.x; qb[hf][5] = b1.y; qb[hf][6] = b1.z; qb[hf][7] = b1.w;
          }
        }
        uint32_t wa[2][8], wb[2][8];
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            float da[2], db[2];
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
              const float a = h2 ? bf16hi(qa[hf][q]) : bf16lo(qa[hf][q]);
              const float b = h2 ? bf16hi(qb[hf][q]) : bf16lo(qb[hf][q]);
              const float dm = u2f(v[16 * hf + 2 * q + h2]);
              // fast division: with the IEEE one this epilogue outlasted the
              // next tile's mainloop at K = 5120 (13B: 1.09 -> 1.3 PFLOP/s)
              const float sg = __fdividef(1.0f, 1.0f + __expf(-a));
              db[h2] = dm * a * sg;
              da[h2] = dm * b * sg * (1.0f + a * (1.0f - sg));
            }
            wa[hf][q] = pack_bf16(da[0], da[1]);
            wb[hf][q] = pack_bf16(db[0], db[1]);
          }
        }
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          __nv_bfloat16* pa_ = arow + f0 + 16 * hf;
          __nv_bfloat16* pb_ = arow + F + f0 + 16 * hf;
          if (v8[hf]) {
            st_global_v8(pa_, wa[hf]);
            st_global_v8(pb_, wb[hf]);
          } else {
            *reinterpret_cast<uint4*>(pa_) = make_uint4(wa[hf][0], wa[hf][1], wa[hf][2], wa[hf][3]);
            *reinterpret_cast<uint4*>(pa_ + 8) = make_uint4(wa[hf][4], wa[hf][5], wa[hf][6], wa[hf][7]);
            *reinterpret_cast<uint4*>(pb_) = make_uint4(wb[hf][0], wb[hf][1], wb[hf][2], wb[hf][3]);
            *reinterpret_cast<uint4*>(pb_ + 8) = make_uint4(wb[hf][4], wb[hf][5], wb[hf][6], wb[hf][7]);
          }
        }
      }
    }
  } else if constexpr (EPI == EPI_CE_STATS) {
    // Pass 1: the row's max (lowest index on ties), argmax and target logit
    // over the tile's 256 columns.  Pass 2: sum exp(S - max) and, when
    // args.ds is set, store P~ = exp(S - max) as fp16 into the dS buffer, so
    // the backward forms dS = coef (P~ exp(max - lse) - onehot) elementwise
    // (launch_ce_ds_from_p) instead of recomputing S with a second GEMM.
    const int yl = row_ok ? args.targets[gm] - args.vocab_begin : -1;
    float mx = -INFINITY, tl = 0.0f;
    int am = 0;
    bool has_t = false;
#pragma unroll 1
    for (int c = 0; c < GEMM_BN / 32; ++c) {
      uint32_t v[32];
      tmem_ld_32x32b_x32(tb + c * 32, v);
      tmem_ld_wait();
      const int gn0 = nb * GEMM_BN + c * 32;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float x = u2f(v[j]);
        if (gn0 + j < args.N && x > mx) {
          mx = x;
          am = gn0 + j;
        }
        if (gn0 + j == yl) {
          tl = x;
          has_t = true;
        }
      }
    }
    float sm = 0.0f;
    __half* prow = (row_ok && args.ds) ? reinterpret_cast<__half*>(args.ds) + (long long)gm * args.ld_ds
                                       : nullptr;
#pragma unroll 1
    for (int c = 0; c < GEMM_BN / 32; ++c) {
      uint32_t v[32];
      tmem_ld_32x32b_x32(tb + c * 32, v);
      tmem_ld_wait();
      const int gn0 = nb * GEMM_BN + c * 32;
      float cs = 0.0f;
#pragma unroll
      for (int j = 0; j < 32; j += 16) {
        uint32_t w[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int c0 = gn0 + j + 2 * q;
          const float e0 = c0 < args.N ? __expf(u2f(v[j + 2 * q]) - mx) : 0.0f;
          const float e1 = c0 + 1 < args.N ? __expf(u2f(v[j + 2 * q + 1]) - mx) : 0.0f;
          cs += e0 + e1;
          const __half2 hp = __floats2half2_rn(e0, e1);
          w[q] = *reinterpret_cast<const uint32_t*>(&hp);
        }
        if (prow != nullptr && gn0 + j < args.N) {
          __half* pd = prow + gn0 + j;
          if (gn0 + j + 16 <= args.N && aligned32(pd)) {
            st_global_v8(pd, w);
          } else {
            *reinterpret_cast<uint4*>(pd) = make_uint4(w[0], w[1], w[2], w[3]);
            if (gn0 + j + 8 < args.N)
              *reinterpret_cast<uint4*>(pd + 8) = make_uint4(w[4], w[5], w[6], w[7]);
          }
        }
      }
      sm += cs;
    }
    if (row_ok) {
      const long long o = (long long)nb * args.M + gm;
      args.part_m[o] = mx;
      args.part_s[o] = sm;
      args.part_i[o] = am + args.vocab_begin;
      if (has_t) args.tgt_logit[gm] = tl;
    }
  } else if constexpr (EPI == EPI_CE_DS) {
    const int yl = row_ok ? args.targets[gm] - args.vocab_begin : -1;
    const float l = row_ok ? args.lse[gm] : 0.0f;
    const float cf = row_ok ? args.coef[gm] : 0.0f;
    __nv_bfloat16* drow = row_ok ? args.ds + (long long)gm * args.ld_ds : nullptr;
#pragma unroll 1
    for (int c = 0; c < GEMM_BN / 32; ++c) {
      uint32_t v[32];
      tmem_ld_32x32b_x32(tb + c * 32, v);
      tmem_ld_wait();
      const int gn0 = nb * GEMM_BN + c * 32;
      if (row_ok && gn0 < args.N) {
#pragma unroll
        for (int j = 0; j < 32; j += 16) {
          if (gn0 + j >= args.N) continue;
          uint32_t w[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int c0 = gn0 + j + 2 * q;
            const float d0 = cf * (__expf(u2f(v[j + 2 * q]) - l) - (c0 == yl ? 1.0f : 0.0f));
            const float d1 =
                cf * (__expf(u2f(v[j + 2 * q + 1]) - l) - (c0 + 1 == yl ? 1.0f : 0.0f));
            w[q] = pack_bf16(d0, d1);
          }
          __nv_bfloat16* pd = drow + gn0 + j;
          if (gn0 + j + 16 <= args.N && aligned32(pd)) {
            st_global_v8(pd, w);
          } else {
            *reinterpret_cast<uint4*>(pd) = make_uint4(w[0], w[1], w[2], w[3]);
            if (gn0 + j + 8 < args.N)
              *reinterpret_cast<uint4*>(pd + 8) = make_uint4(w[4], w[5], w[6], w[7]);
          }
        }
      }
    }
  }
}

template <int EPI, bool A_MN, bool B_MN>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB0,
                const __grid_constant__ CUtensorMap tmB1, const GemmArgs args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + GEMM_STAGES * GEMM_A_STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + GEMM_STAGES * GEMM_B_STAGE);
  uint64_t* empty = full + GEMM_STAGES;
  uint64_t* tfull = empty + GEMM_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB0);
    if (args.b_mode != B_PLAIN) tma_prefetch_desc(&tmB1);
    for (int s = 0; s < GEMM_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 128);
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    tmem_alloc(tmem_slot, GEMM_TMEM_COLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int num_tiles = args.m_blocks * args.n_blocks;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      const uint64_t pa = l2_policy(args.hint_a), pb = l2_policy(args.hint_b);
      const bool ha = args.hint_a >= 0, hb = args.hint_b >= 0;
      auto lda = [&](void* d, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
        if (ha) tma_load_2d_hint(d, m, bar, c0, c1, pa); else tma_load_2d(d, m, bar, c0, c1);
      };
      auto ldb = [&](void* d, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
        if (hb) tma_load_2d_hint(d, m, bar, c0, c1, pb); else tma_load_2d(d, m, bar, c0, c1);
      };
      int s = 0;
      uint32_t ph = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        int mb, nb;
        tile_coords(args, tile, mb, nb);
        const int m0 = mb * GEMM_BM;
        for (int kb = 0; kb < args.k_blocks; ++kb) {
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t* a = sA + s * GEMM_A_STAGE;
          uint8_t* b = sB + s * GEMM_B_STAGE;
          const int k0 = kb * GEMM_BK;
          if constexpr (!A_MN) {
            lda(a, &tmA, &full[s], k0, m0);
          } else {
            lda(a, &tmA, &full[s], m0, k0);
            lda(a + 8192, &tmA, &full[s], m0 + 64, k0);
          }
          if (args.b_mode == B_PAIR) {
            const int n0 = nb * (GEMM_BN / 2);
            ldb(b, &tmB0, &full[s], k0, n0);
            ldb(b + GEMM_B_STAGE / 2, &tmB1, &full[s], k0, n0);
          } else {
            const CUtensorMap* mB = &tmB0;
            int kk = k0;
            if (args.b_mode == B_KSPLIT && k0 >= args.b_ksplit) {
              mB = &tmB1;
              kk = k0 - args.b_ksplit;
            }
            const int n0 = nb * GEMM_BN;
            if constexpr (!B_MN) {
              ldb(b, mB, &full[s], kk, n0);
            } else {
#pragma unroll
              for (int j = 0; j < 4; ++j) ldb(b + j * 8192, mB, &full[s], n0 + 64 * j, kk);
            }
          }
          mbar_arrive_expect_tx(&full[s], GEMM_A_STAGE + GEMM_B_STAGE);
          if (++s == GEMM_STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc_bf16(GEMM_BM, GEMM_BN, A_MN, B_MN);
      int s = 0;
      uint32_t ph = 0;
      int acc = 0;
      uint32_t acc_ph = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        mbar_wait(&tempty[acc], acc_ph ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * GEMM_BN;
        for (int kb = 0; kb < args.k_blocks; ++kb) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + s * GEMM_A_STAGE);
          const uint32_t b_addr = smem_u32(sB + s * GEMM_B_STAGE);
#pragma unroll
          for (int k = 0; k < GEMM_BK / 16; ++k) {
            const uint64_t ad = A_MN ? make_sdesc(a_addr + k * 2048, 8192, 1024)
                                     : make_sdesc(a_addr + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? make_sdesc(b_addr + k * 2048, 8192, 1024)
                                     : make_sdesc(b_addr + k * 32, 16, 1024);
            tc_mma_f16(d_tmem, ad, bd, idesc, (kb | k) != 0 ? 1u : 0u);
          }
          tc_commit(&empty[s]);
          if (++s == GEMM_STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
        tc_commit(&tfull[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_ph ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    const int ew = warp - 4;  // == warp % 4: TMEM lanes [32*ew, 32*ew+32)
    const int row = ew * 32 + lane;
    int acc = 0;
    uint32_t acc_ph = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      int mb, nb;
      tile_coords(args, tile, mb, nb);
      const int gm = mb * GEMM_BM + row;
      const bool row_ok = gm < args.M;
      if (args.epi_sleep >= 2)
        mbar_wait_backoff(&tfull[acc], acc_ph, (uint32_t)args.epi_sleep);
      else if (args.epi_sleep)
        mbar_wait_sleep(&tfull[acc], acc_ph);
      else
        mbar_wait(&tfull[acc], acc_ph);
      tc_fence_after();
      const uint32_t tb = tmem_base + acc * GEMM_BN + (static_cast<uint32_t>(ew * 32) << 16);
      if (args.trace && threadIdx.x == 128) args.trace[tile] = trace_stamp();
      (void)row_ok;
      epilogue_tile<EPI>(args, tb, gm, nb);
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_ph ^= 1;
      }
    }
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, GEMM_TMEM_COLS);
  }
}


// ============================================================================
// CTA-pair variant (tcgen05 cta_group::2): a cluster of 2 CTAs on the two SMs
// of a TPC computes a 256 x 256 tile.  Each CTA stages its own 128 rows of A
// and its own 128-row half of B (N) per stage; the leader's single thread
// issues tcgen05.mma.cta_group::2 (M = 256) which reads both CTAs' smem and
// writes each CTA's 128 accumulator rows into that CTA's TMEM.  Per SM this
// halves the B bytes pulled from L2 and read from smem per FLOP versus the
// 128 x 256 single-CTA tile.
//   - full[s]   lives in the leader; both CTAs' TMA (cta_group::2 form) count
//               their bytes on it; only the leader's MMA thread waits on it.
//   - empty[s]  in both CTAs; the leader's tcgen05.commit multicasts to both.
//   - tfull[a]  in both CTAs (multicast commit); tempty[a] in the leader,
//               256 arrivals (128 epilogue threads of each CTA, remote via mapa).
// ============================================================================
// NB2 = 256-column accumulator halves per pair tile: 1 -> 256 x 256 tiles with a
// double-buffered accumulator (2 x 256 TMEM columns); 2 -> 256 x 512 tiles, one
// accumulator filling all 512 columns (no epilogue overlap, but 25% fewer
// operand bytes per FLOP from L2 and DRAM: used for the long-K GEMMs).
template <int NB2>
struct G2Cfg {
  static constexpr int STAGES = NB2 == 1 ? 6 : 4;
  static constexpr int A_STAGE = 128 * GEMM_BK * 2;        // 16 KB: this CTA's 128 rows of A
  static constexpr int B_STAGE = NB2 * 128 * GEMM_BK * 2;  // this CTA's NB2 x 128 rows of B
  static constexpr int NACC = NB2 == 1 ? 2 : 1;            // accumulator buffers in TMEM
  static constexpr int TILE_N = NB2 * GEMM_BN;
  static constexpr int SMEM = STAGES * (A_STAGE + B_STAGE) + 1024 + 256;
};
constexpr int G2_SQ = 4;  // depth of the tile-index ring (dynamic schedule)
constexpr int G2_SMEM = G2Cfg<1>::SMEM;

template <int EPI, bool A_MN, bool B_MN, int NB2 = 1>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(GEMM_THREADS, 1)
    gemm2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB0,
                 const __grid_constant__ CUtensorMap tmB1, const GemmArgs args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  using C = G2Cfg<NB2>;
  constexpr int G2_STAGES = C::STAGES;
  constexpr int G2_A_STAGE = C::A_STAGE;
  constexpr int G2_B_STAGE = C::B_STAGE;
  uint8_t* sA = smem;
  uint8_t* sB = smem + G2_STAGES * G2_A_STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + G2_STAGES * G2_B_STAGE);
  uint64_t* empty = full + G2_STAGES;
  uint64_t* tfull = empty + G2_STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* sfull = tempty + 2;        // tile ring: slot published (both CTAs)
  uint64_t* sempty = sfull + G2_SQ;     // tile ring: slot consumed (leader, 10 arrivals)
  int* ring = reinterpret_cast<int*>(sempty + G2_SQ);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ring + G2_SQ);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int cluster_id = blockIdx.x >> 1;
  const int nclusters = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB0);
    if (args.b_mode != B_PLAIN) tma_prefetch_desc(&tmB1);
    for (int s = 0; s < G2_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 256);
    }
    for (int s = 0; s < G2_SQ; ++s) {
      mbar_init(&sfull[s], 1);
      mbar_init(&sempty[s], 10);  // leader MMA + 4 epilogue warps of each CTA + peer producer
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    tmem_alloc_2sm(tmem_slot, GEMM_TMEM_COLS);
    tmem_relinquish_2sm();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int num_tiles = args.m_blocks * args.n_blocks;

  // Tile schedule.  Static: cluster c takes tiles c, c+P, ...  Dynamic
  // (args.tile_counter): the leader's producer claims the next tile with an
  // atomicAdd and publishes it through a small smem ring in both CTAs; every
  // consumer unit (leader MMA thread, 4 epilogue warps per CTA, peer producer)
  // reads it and releases the slot.  Clusters then take tiles in global order
  // as they free up, so the clusters sharing an operand block stay within a
  // tile of each other instead of drifting apart over hundreds of tiles (the
  // drift cost 3x DRAM traffic: profiles/r01_cta2_trace.log).
  const bool dyn = args.tile_counter != nullptr;
  int sj = 0;
  uint32_t sph = 0;
  auto take = [&]() -> int {  // one lane per consumer unit
    mbar_wait_acq_cluster(&sfull[sj], sph);
    const int t = ring[sj];
    if (leader)
      mbar_arrive(&sempty[sj]);
    else
      mbar_arrive_cluster(mapa_shared(smem_u32(&sempty[sj]), 0));
    if (++sj == G2_SQ) {
      sj = 0;
      sph ^= 1;
    }
    return t;
  };
  auto publish = [&]() -> int {  // leader producer
    mbar_wait(&sempty[sj], sph ^ 1);
    int t = atomicAdd(args.tile_counter, 1);
    if (t >= num_tiles) t = -1;
    ring[sj] = t;
    st_shared_cluster_u32(mapa_shared(smem_u32(&ring[sj]), 1), (uint32_t)t);
    mbar_arrive(&sfull[sj]);
    mbar_arrive_cluster(mapa_shared(smem_u32(&sfull[sj]), 1));
    if (++sj == G2_SQ) {
      sj = 0;
      sph ^= 1;
    }
    return t;
  };
  auto first_tile = [&](bool producer) -> int {
    if (!dyn) return cluster_id;
    return producer ? (leader ? publish() : take()) : take();
  };
  auto next_tile = [&](int tile, bool producer) -> int {
    if (!dyn) return tile + nclusters;
    return producer ? (leader ? publish() : take()) : take();
  };

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    if (lane == 0) {
      const uint64_t pa = l2_policy(args.hint_a), pb = l2_policy(args.hint_b);
      const bool ha = args.hint_a >= 0, hb = args.hint_b >= 0;
      auto lda = [&](void* d, const CUtensorMap* m, uint32_t bar, int c0, int c1) {
        if (ha) tma_load_2d_2sm_hint(d, m, bar, c0, c1, pa); else tma_load_2d_2sm(d, m, bar, c0, c1);
      };
      auto ldb = [&](void* d, const CUtensorMap* m, uint32_t bar, int c0, int c1) {
        if (hb) tma_load_2d_2sm_hint(d, m, bar, c0, c1, pb); else tma_load_2d_2sm(d, m, bar, c0, c1);
      };
      int s = 0;
      uint32_t ph = 0;
      int wave = 0;
      for (int tile = first_tile(true); tile >= 0 && tile < num_tiles;
           tile = next_tile(tile, true), ++wave) {
        if (args.wave_counter != nullptr && leader) {
          // Soft wave barrier (static schedule): the leaders of all clusters
          // start wave w together, so clusters sharing an operand stream the
          // same K range at the same time and hit in L2 (long-K GEMMs).  The
          // wait is bounded (50 us) so co-running kernels (NCCL) that keep a
          // cluster off the GPU cannot deadlock it.
          red_add_release_gpu(args.wave_counter, 1);
          const int target = min(num_tiles, (wave + 1) * nclusters);
          const unsigned long long t0 = globaltimer_ns();
          while (ld_acquire_gpu(args.wave_counter) < target &&
                 globaltimer_ns() - t0 < 50000ull) {
          }
        }
        int mb, nb;
        tile_coords(args, tile, mb, nb);
        const int m0 = mb * 256 + (int)rank * 128;
        for (int kb = 0; kb < args.k_blocks; ++kb) {
          mbar_wait(&empty[s], ph ^ 1);
          const uint32_t fb = mapa_shared(smem_u32(&full[s]), 0);
          uint8_t* a = sA + s * G2_A_STAGE;
          uint8_t* b = sB + s * G2_B_STAGE;
          const int k0 = kb * GEMM_BK;
          if constexpr (!A_MN) {
            lda(a, &tmA, fb, k0, m0);
          } else {
            lda(a, &tmA, fb, m0, k0);
            lda(a + 8192, &tmA, fb, m0 + 64, k0);
          }
          if (args.b_mode == B_PAIR) {
            // CTA 0 holds the 128 gate rows, CTA 1 the 128 up rows of the same f range
            ldb(b, rank ? &tmB1 : &tmB0, fb, k0, nb * 128);
          } else {
            const CUtensorMap* mB = &tmB0;
            int kk = k0;
            if (args.b_mode == B_KSPLIT && k0 >= args.b_ksplit) {
              mB = &tmB1;
              kk = k0 - args.b_ksplit;
            }
#pragma unroll
            for (int hh = 0; hh < NB2; ++hh) {
              // half hh of the pair tile: columns [n0h, n0h + 256), CTA r holds rows
              // n0h + 128 r .. +128 in smem rows [128 hh, 128 hh + 128)
              const int n0 = nb * C::TILE_N + hh * GEMM_BN + (int)rank * 128;
              uint8_t* bh = b + hh * 16384;
              if constexpr (!B_MN) {
                ldb(bh, mB, fb, kk, n0);
              } else {
                ldb(bh, mB, fb, n0, kk);
                ldb(bh + 8192, mB, fb, n0 + 64, kk);
              }
            }
          }
          if (leader) mbar_arrive_expect_tx(&full[s], 2 * (G2_A_STAGE + G2_B_STAGE));
          if (++s == G2_STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader only)
    // The whole warp runs the loop (descriptors in uniform registers) and
    // elect.sync issues each tcgen05 instruction; lane 0 alone consumes the
    // tile schedule and broadcasts it.
    if (leader) {
      constexpr uint32_t idesc = make_idesc_bf16(256, GEMM_BN, A_MN, B_MN);
      int s = 0;
      uint32_t ph = 0;
      int acc = 0;
      uint32_t acc_ph = 0;
      auto mma_tile = [&](int prev, bool first) -> int {
        int t = 0;
        if (lane == 0) t = first ? first_tile(false) : next_tile(prev, false);
        return __shfl_sync(0xffffffffu, t, 0);
      };
      for (int tile = mma_tile(0, true); tile >= 0 && tile < num_tiles;
           tile = mma_tile(tile, false)) {
        mbar_wait(&tempty[acc], acc_ph ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * GEMM_BN;
        for (int kb = 0; kb < args.k_blocks; ++kb) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + s * G2_A_STAGE);
          const uint32_t b_addr = smem_u32(sB + s * G2_B_STAGE);
#pragma unroll
          for (int k = 0; k < GEMM_BK / 16; ++k) {
            const uint64_t ad = A_MN ? make_sdesc(a_addr + k * 2048, 8192, 1024)
                                     : make_sdesc(a_addr + k * 32, 16, 1024);
#pragma unroll
            for (int hh = 0; hh < NB2; ++hh) {
              const uint32_t bh = b_addr + hh * 16384;
              const uint64_t bd = B_MN ? make_sdesc(bh + k * 2048, 8192, 1024)
                                       : make_sdesc(bh + k * 32, 16, 1024);
              tc_mma_f16_2sm_w(d_tmem + hh * GEMM_BN, ad, bd, idesc, (kb | k) != 0 ? 1u : 0u);
            }
          }
          tc_commit_2sm_w(&empty[s], 0x3);
          if (++s == G2_STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
        tc_commit_2sm_w(&tfull[acc], 0x3);
        if (++acc == C::NACC) {
          acc = 0;
          acc_ph ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue (both CTAs)
    const int ew = warp - 4;
    const int row = ew * 32 + lane;
    int acc = 0;
    uint32_t acc_ph = 0;
    const uint32_t te0 = mapa_shared(smem_u32(&tempty[0]), 0);
    const uint32_t te1 = mapa_shared(smem_u32(&tempty[1]), 0);
    auto warp_tile = [&](int prev, bool first) -> int {  // lane 0 consumes, broadcast
      int t = 0;
      if (lane == 0) t = first ? first_tile(false) : next_tile(prev, false);
      return __shfl_sync(0xffffffffu, t, 0);
    };
    for (int tile = warp_tile(0, true); tile >= 0 && tile < num_tiles;
         tile = warp_tile(tile, false)) {
      int mb, nb;
      tile_coords(args, tile, mb, nb);
      if constexpr (EPI == EPI_F32T && NB2 == 1) {
        // gain identity (A28): this tile's epilogue reads W[n][m] for its 256
        // columns n and this CTA's 128 rows m (256 B per row).  Prefetch them
        // into L2 while the mainloop runs: read cold, the 64-byte pieces at a
        // 16 KB stride exposed DRAM latency chunk by chunk and at K = 8192 (DP
        // over 8 ranks) the epilogue outlasted the mainloop 4x (profiles/r02dp8)
        if (args.gain_part != nullptr && lane == 0) {
          const int m0 = mb * 256 + (int)rank * 128;
          if (m0 < args.M) {
            const uint32_t bytes = (uint32_t)(min(128, args.M - m0) * 2);
            for (int i = ew; i < GEMM_BN; i += 4) {
              const int gn = nb * GEMM_BN + i;
              if (gn >= args.N) break;
              const __nv_bfloat16* w = gn < args.n_split
                                           ? args.gain_w0 + (long long)gn * args.M + m0
                                           : args.gain_w1 + (long long)(gn - args.n_split) * args.M + m0;
              bulk_prefetch_l2(w, bytes);
            }
          }
        }
      }
      if (args.epi_sleep >= 2)
        mbar_wait_backoff(&tfull[acc], acc_ph, (uint32_t)args.epi_sleep);
      else if (args.epi_sleep)
        mbar_wait_sleep(&tfull[acc], acc_ph);
      else
        mbar_wait(&tfull[acc], acc_ph);
      tc_fence_after();
      const uint32_t tb = tmem_base + acc * GEMM_BN + (static_cast<uint32_t>(ew * 32) << 16);
      if (args.trace && threadIdx.x == 128 && rank == 0) args.trace[tile] = trace_stamp();
#pragma unroll 1
      for (int hh = 0; hh < NB2; ++hh)
        // a 512-wide tile's second half may lie past N (NB2 = 2 only: with B_PAIR
        // the tile columns are 128 + 128 of two matrices and N counts one of them)
        if (NB2 == 1 || (nb * NB2 + hh) * GEMM_BN < args.N)
          epilogue_tile<EPI>(args, tb + hh * GEMM_BN, mb * 256 + (int)rank * 128 + row,
                             nb * NB2 + hh);
      tc_fence_before();
      mbar_arrive_cluster(acc ? te1 : te0);
      if (++acc == C::NACC) {
        acc = 0;
        acc_ph ^= 1;
      }
    }
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_2sm(tmem_base, GEMM_TMEM_COLS);
  }
}

}  // namespace ee
