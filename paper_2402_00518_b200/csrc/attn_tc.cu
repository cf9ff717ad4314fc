// attn_tc.cu -- causal GQA flash-attention forward on the 5th-generation
// tensor cores (tcgen05 + TMEM + TMA) for the Layer exit and the backbone
// (Llama-2 attention; Layer exit P:210).
//
// One CTA per (128-query tile, query head, sequence); head dim 128.
//   warp 0      TMA producer: Q once, then K_j / V_j (128 keys) into a 2-stage ring
//   warp 1      MMA issuer (one thread): S_j = Q K_j^T into one of two TMEM
//               S buffers, then O (+)= P_j V_j into the TMEM O accumulator
//   warps 4..7  softmax, one thread per query row (= TMEM lane): reads S_j,
//               keeps the running max m and sum l in registers, writes
//               P_j = 2^(s log2e/sqrt(d) - m) as bf16 into shared memory in the
//               SWIZZLE_128B K-major layout the MMA reads as its A operand;
//               finally O / l -> bf16 and lse2 = m + log2 l.
// The MMA of S_{j+1} runs while the softmax threads work on S_j.  O lives in
// TMEM for the whole key loop; it is rescaled (TMEM ld/st) only when a row's
// max grows by more than 2^8 over the reference max used so far -- with a
// fixed reference m, O / l is exact whatever m is, and P stays <= 2^8 in bf16.
// Causal mask on the diagonal tile only (key > query); tiles past a short
// sequence's end are excluded by the same mask, so T need only be a multiple
// of 64.  Heavy (late) query tiles are scheduled first.
#include <cmath>
#include "internal.cuh"

namespace ee {

namespace {
constexpr int FA_BM = 128;                        // queries per CTA
constexpr int FA_BN = 128;                        // keys per tile
constexpr int FA_D = 128;                         // head dim
constexpr int FA_TILE = FA_BM * FA_D * 2;         // 32 KB: two 16 KB SW128 atoms
constexpr int FA_ATOM = 16384;
constexpr int FA_STAGES = 2;
constexpr int FA_SMEM = 1024 + FA_TILE * (2 + 2 * FA_STAGES) + 256;
constexpr float FA_RESCALE = 8.0f;                // log2 headroom before O is rescaled
}  // namespace

__global__ void __launch_bounds__(256, 1)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                       const __grid_constant__ CUtensorMap tmV, __nv_bfloat16* __restrict__ o,
                       float* __restrict__ lse2, int T, int Hq, int Hkv, float scale_log2) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + FA_TILE;
  uint8_t* sV = sK + FA_STAGES * FA_TILE;
  uint8_t* sP = sV + FA_STAGES * FA_TILE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + FA_TILE);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;   // [2]
  uint64_t* kv_empty = bars + 3;  // [2]
  uint64_t* s_full = bars + 5;    // [2]
  uint64_t* p_full = bars + 7;
  uint64_t* o_done = bars + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 9);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqt = (T + FA_BM - 1) / FA_BM;
  const int qt = nqt - 1 - (int)blockIdx.x;  // longest causal rows first
  const int hq = blockIdx.y, b = blockIdx.z;
  const int hk = hq / (Hq / Hkv);
  const int q_row0 = b * T + qt * FA_BM;
  const int n_kt = qt + 1;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    mbar_init(q_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
      mbar_init(&s_full[s], 1);
    }
    mbar_init(p_full, 128);
    mbar_init(o_done, 1);
    fence_barrier_init();
  }
  if (warp == 2) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t tS0 = tmem_base, tO = tmem_base + 2 * FA_BN;

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      tma_load_2d(sQ, &tmQ, q_full, hq * FA_D, q_row0);
      tma_load_2d(sQ + FA_ATOM, &tmQ, q_full, hq * FA_D + 64, q_row0);
      mbar_arrive_expect_tx(q_full, FA_TILE);
      for (int j = 0; j < n_kt; ++j) {
        const int s = j & 1;
        mbar_wait(&kv_empty[s], ((j >> 1) & 1) ^ 1);
        const int k_row0 = b * T + j * FA_BN;
        uint8_t* k = sK + s * FA_TILE;
        uint8_t* v = sV + s * FA_TILE;
        tma_load_2d(k, &tmK, &kv_full[s], hk * FA_D, k_row0);
        tma_load_2d(k + FA_ATOM, &tmK, &kv_full[s], hk * FA_D + 64, k_row0);
        tma_load_2d(v, &tmV, &kv_full[s], hk * FA_D, k_row0);
        tma_load_2d(v + FA_ATOM, &tmV, &kv_full[s], hk * FA_D + 64, k_row0);
        mbar_arrive_expect_tx(&kv_full[s], 2 * FA_TILE);
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc_qk = make_idesc_bf16(FA_BM, FA_BN, false, false);
      constexpr uint32_t idesc_pv = make_idesc_bf16(FA_BM, FA_D, false, true);
      const uint32_t aq = smem_u32(sQ), ap = smem_u32(sP);
      mbar_wait(q_full, 0);
      auto issue_qk = [&](int j) {
        const int s = j & 1;
        mbar_wait(&kv_full[s], (j >> 1) & 1);
        tc_fence_after();
        const uint32_t bk = smem_u32(sK + s * FA_TILE);
#pragma unroll
        for (int k = 0; k < FA_D / 16; ++k) {  // K-major A and B: 4 k-steps per 64-wide atom
          const uint32_t off = (k >> 2) * FA_ATOM + (k & 3) * 32;
          tc_mma_f16(tS0 + s * FA_BN, make_sdesc(aq + off, 16, 1024), make_sdesc(bk + off, 16, 1024),
                     idesc_qk, k != 0 ? 1u : 0u);
        }
        tc_commit(&s_full[s]);
      };
      issue_qk(0);
      for (int j = 0; j < n_kt; ++j) {
        if (j + 1 < n_kt) issue_qk(j + 1);
        mbar_wait(p_full, j & 1);
        tc_fence_after();
        const uint32_t bv = smem_u32(sV + (j & 1) * FA_TILE);
#pragma unroll
        for (int k = 0; k < FA_BN / 16; ++k) {  // A = P (K-major), B = V (MN-major: keys x d)
          const uint32_t offa = (k >> 2) * FA_ATOM + (k & 3) * 32;
          tc_mma_f16(tO, make_sdesc(ap + offa, 16, 1024), make_sdesc(bv + k * 2048, FA_ATOM, 1024),
                     idesc_pv, (j | k) != 0 ? 1u : 0u);
        }
        tc_commit(o_done);
        tc_commit(&kv_empty[j & 1]);
      }
    }
  } else if (warp >= 4) {
    // ---------------------------------------------------------------- softmax
    const int ew = warp - 4;
    const int r = ew * 32 + lane;  // query row within the tile = TMEM lane
    const uint32_t lane_off = static_cast<uint32_t>(ew * 32) << 16;
    float m_ref = -INFINITY, l = 0.f;
    uint8_t* prow = sP + r * 128;
    for (int j = 0; j < n_kt; ++j) {
      mbar_wait(&s_full[j & 1], (j >> 1) & 1);
      tc_fence_after();
      float sv[FA_BN];
      const uint32_t ts = tS0 + (j & 1) * FA_BN + lane_off;
#pragma unroll
      for (int c = 0; c < FA_BN / 32; ++c) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(ts + c * 32, v);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) sv[c * 32 + i] = __uint_as_float(v[i]) * scale_log2;
      }
      if (j == qt) {  // diagonal tile: key column > query row is in the future
#pragma unroll
        for (int i = 0; i < FA_BN; ++i)
          if (i > r) sv[i] = -INFINITY;
      }
      float mx = sv[0];
#pragma unroll
      for (int i = 1; i < FA_BN; ++i) mx = fmaxf(mx, sv[i]);
      if (j > 0) {
        mbar_wait(o_done, (j - 1) & 1);  // PV_{j-1} done: O stable, P buffer free
        tc_fence_after();
      }
      if (j == 0) {
        m_ref = mx;
      } else {
        // tcgen05.ld/st are warp-collective: the rescale decision is per warp
        // (rows that did not grow past the headroom use alpha = 1)
        const bool grow = mx > m_ref + FA_RESCALE;
        if (__any_sync(0xffffffffu, grow)) {
          const float alpha = grow ? ex2_approx(m_ref - mx) : 1.0f;
          if (grow) {
            l *= alpha;
            m_ref = mx;
          }
#pragma unroll 1
          for (int c = 0; c < FA_D / 32; ++c) {
            uint32_t v[32];
            tmem_ld_32x32b_x32(tO + lane_off + c * 32, v);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * alpha);
            tmem_st_32x32b_x32(tO + lane_off + c * 32, v);
          }
          tmem_st_wait();
        }
      }
      // P = 2^(s - m_ref) -> bf16, K-major SWIZZLE_128B: 16-byte chunk cc of
      // row r sits at chunk (cc ^ (r & 7)) of the row's 128-byte line
#pragma unroll
      for (int c8 = 0; c8 < FA_BN / 8; ++c8) {
        float p[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          p[e] = ex2_approx(sv[c8 * 8 + e] - m_ref);
          l += p[e];
        }
        const uint4 w = make_uint4(pack_bf16(p[0], p[1]), pack_bf16(p[2], p[3]),
                                   pack_bf16(p[4], p[5]), pack_bf16(p[6], p[7]));
        const int cc = c8 & 7;
        *reinterpret_cast<uint4*>(prow + (c8 >> 3) * FA_ATOM + ((cc ^ (r & 7)) << 4)) = w;
      }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(p_full);
    }
    // ---------------------------------------------------------------- epilogue
    mbar_wait(o_done, (n_kt - 1) & 1);
    tc_fence_after();
    const int pos = qt * FA_BM + r;
    const bool ok = pos < T;
    const float inv_l = 1.0f / l;
    __nv_bfloat16* orow = o + (long long)(q_row0 + r) * Hq * FA_D + hq * FA_D;
#pragma unroll 1
    for (int c = 0; c < FA_D / 32; ++c) {
      uint32_t v[32];
      tmem_ld_32x32b_x32(tO + lane_off + c * 32, v);
      tmem_ld_wait();
      if (ok) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t w[8];
#pragma unroll
          for (int q = 0; q < 8; ++q)
            w[q] = pack_bf16(__uint_as_float(v[h * 16 + 2 * q]) * inv_l,
                             __uint_as_float(v[h * 16 + 2 * q + 1]) * inv_l);
          __nv_bfloat16* dst = orow + c * 32 + h * 16;
          if (aligned32(dst)) {
            st_global_v8(dst, w);
          } else {
            *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
            *reinterpret_cast<uint4*>(dst + 8) = make_uint4(w[4], w[5], w[6], w[7]);
          }
        }
      }
    }
    if (ok && lse2 != nullptr) lse2[(long long)(q_row0 + r) * Hq + hq] = m_ref + log2f(l);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

cudaError_t launch_attn_fwd_tc(const __nv_bfloat16* q, const __nv_bfloat16* k,
                               const __nv_bfloat16* v, __nv_bfloat16* o, long long N, int T,
                               int Hq, int Hkv, float* lse2, cudaStream_t s) {
  if (N == 0) return cudaSuccess;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_fwd_tc_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, FA_SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  CUtensorMap tq, tk, tv;
  const Mat Q{q, N, (long long)Hq * FA_D, (long long)Hq * FA_D};
  const Mat K{k, N, (long long)Hkv * FA_D, (long long)Hkv * FA_D};
  const Mat V{v, N, (long long)Hkv * FA_D, (long long)Hkv * FA_D};
  if (!make_tmap(&tq, Q, 64, FA_BM) || !make_tmap(&tk, K, 64, FA_BN) || !make_tmap(&tv, V, 64, FA_BN))
    return cudaErrorInvalidValue;
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)FA_D);
  dim3 grid((T + FA_BM - 1) / FA_BM, Hq, (unsigned)(N / T));
  attn_fwd_tc_kernel<<<grid, 256, FA_SMEM, s>>>(tq, tk, tv, o, lse2, T, Hq, Hkv, scale_log2);
  return cudaGetLastError();
}

}  // namespace ee
