// gemm.cu -- host side of the tcgen05 GEMM: TMA descriptors and dispatch.
#include <atomic>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdlib>
#include <mutex>
#include "internal.cuh"

namespace ee {

typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                      const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                      const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                      CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled_t encode_fn() {
  static PFN_encodeTiled_t fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled_t>(p);
  });
  return fn;
}

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// 2-D bf16 tensor map, 128B swizzle; inner = contiguous dim.
bool make_tmap(CUtensorMap* m, const Mat& t, uint32_t box_inner, uint32_t box_outer) {
  PFN_encodeTiled_t enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)t.cols, (cuuint64_t)t.rows};
  cuuint64_t strides[1] = {(cuuint64_t)t.ld * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(t.ptr), dims, strides,
                   box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Per-launch tile counters of the dynamic schedule (CTA-pair kernel): slot k is
// zeroed on the launch's stream right before the launch that uses it.
constexpr int kTileCounters = 4096;
__device__ int g_tile_ctr[kTileCounters];
// Thread-safe: several host threads (ranks sharing a process, or one stream
// per thread) may launch concurrently; a slot is reused only after 4096 launches.
static int* tile_counter(cudaStream_t st) {
  static std::atomic<int*> base{nullptr};
  static std::atomic<unsigned> next{0};
  int* b = base.load();
  if (!b) {
    if (cudaGetSymbolAddress((void**)&b, g_tile_ctr) != cudaSuccess) return nullptr;
    base.store(b);
  }
  int* c = b + (next.fetch_add(1) % kTileCounters);
  if (cudaMemsetAsync(c, 0, sizeof(int), st) != cudaSuccess) return nullptr;
  return c;
}

template <int EPI, bool A_MN, bool B_MN, int NB2 = 1>
static cudaError_t launch2(const CUtensorMap& a, const CUtensorMap& b0, const CUtensorMap& b1,
                           const GemmArgs& args, cudaStream_t st) {
  auto kern = gemm2_kernel<EPI, A_MN, B_MN, NB2>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         G2Cfg<NB2>::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int tiles = args.m_blocks * args.n_blocks;
  const int pairs = num_sms() / 2;
  const int grid = 2 * (tiles < pairs ? tiles : pairs);
  GemmArgs a2 = args;
  // Schedule: K = h GEMMs (short mainloop) take tiles dynamically; long-K
  // GEMMs use the static schedule with a per-wave soft barrier.
  static const int dyn = getenv("EE_GEMM_DYN") ? atoi(getenv("EE_GEMM_DYN")) : 1;
  static const int wsync = getenv("EE_GEMM_WAVESYNC") ? atoi(getenv("EE_GEMM_WAVESYNC")) : 1;
  const bool long_k = args.K >= 16384 || wsync == 2;
  a2.tile_counter = (dyn && !(wsync && long_k)) ? tile_counter(st) : nullptr;
  a2.wave_counter = (wsync && long_k && a2.tile_counter == nullptr) ? tile_counter(st) : nullptr;
  kern<<<grid, GEMM_THREADS, G2Cfg<NB2>::SMEM, st>>>(a, b0, b1, a2);
  return cudaGetLastError();
}

static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

// Debug tile trace (EE_GEMM_TRACE=1): the first GEMM launch after
// ee_debug_trace_arm() records, per tile, when its accumulator became ready.
static unsigned long long* g_trace = nullptr;
static int g_trace_cap = 0, g_trace_n = 0;
static bool g_trace_armed = false;
unsigned long long* trace_buffer(int tiles) {
  if (!g_trace_armed) return nullptr;
  g_trace_armed = false;
  if (tiles > g_trace_cap) {
    if (g_trace) cudaFree(g_trace);
    cudaMalloc(&g_trace, sizeof(unsigned long long) * tiles);
    g_trace_cap = tiles;
  }
  g_trace_n = tiles;
  return g_trace;
}
void debug_trace_arm() { g_trace_armed = true; }
int debug_trace_read(unsigned long long* host, int max) {
  const int n = g_trace_n < max ? g_trace_n : max;
  if (g_trace && n > 0) cudaMemcpy(host, g_trace, sizeof(unsigned long long) * n, cudaMemcpyDeviceToHost);
  return n;
}

template <int EPI, bool A_MN, bool B_MN>
static cudaError_t launch(const CUtensorMap& a, const CUtensorMap& b0, const CUtensorMap& b1,
                          const GemmArgs& args, cudaStream_t st) {
  auto kern = gemm_kernel<EPI, A_MN, B_MN>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, GEMM_SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int tiles = args.m_blocks * args.n_blocks;
  const int grid = tiles < num_sms() ? tiles : num_sms();
  static const int cluster = env_int("EE_GEMM_CLUSTER", 1);  // placement experiment only
  if (cluster > 1 && grid % cluster == 0) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(GEMM_THREADS);
    cfg.dynamicSmemBytes = GEMM_SMEM;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cluster;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, a, b0, b1, args);
  }
  kern<<<grid, GEMM_THREADS, GEMM_SMEM, st>>>(a, b0, b1, args);
  return cudaGetLastError();
}

unsigned long long* trace_buffer(int tiles);
cudaError_t gemm_run(int epi, bool a_kmajor, bool b_kmajor, const Mat& A, const Mat& B0,
                     const Mat* B1, int b_mode, int b_ksplit, GemmArgs args, cudaStream_t st) {
  static const int cta_pair = env_int("EE_GEMM_CTA", 2) == 2;  // CTA pair + dynamic schedule: measured fastest (profiles/r01_cta2_dyn.log)
  static const int group = env_int("EE_GEMM_GROUP", 0);
  static const int hint_a = env_int("EE_GEMM_HINT_A", -1);
  static const int hint_b = env_int("EE_GEMM_HINT_B", -1);
  static const int epi_sleep = env_int("EE_GEMM_SLEEP", 1);
  CUtensorMap ta, tb0, tb1;
  const bool a_mn = !a_kmajor, b_mn = !b_kmajor;
  if (!make_tmap(&ta, A, 64, a_mn ? 64 : GEMM_BM)) return cudaErrorInvalidValue;
  const uint32_t b_outer =
      b_mn ? 64 : ((b_mode == B_PAIR || cta_pair) ? GEMM_BN / 2 : GEMM_BN);
  if (!make_tmap(&tb0, B0, 64, b_outer)) return cudaErrorInvalidValue;
  if (b_mode != B_PLAIN) {
    if (!B1 || !make_tmap(&tb1, *B1, 64, b_outer)) return cudaErrorInvalidValue;
  } else {
    tb1 = tb0;
  }
  args.b_mode = b_mode;
  args.b_ksplit = b_ksplit;
  const int bm = cta_pair ? 2 * GEMM_BM : GEMM_BM;
  args.m_blocks = (args.M + bm - 1) / bm;
  // 256 x 512 pair tiles for the long-K GEMMs (EE_GEMM_WIDE=1): 25% fewer
  // operand bytes per FLOP on paper, but measured 7% slower per step at the
  // power cap (profiles/r01_wide_ab.log), so off by default
  static const int wide_env = env_int("EE_GEMM_WIDE", 0);  // measured slower (profiles/r01_wide_ab.log); 2: any K (experiment)
  const bool wide = cta_pair && wide_env && b_mode != B_PAIR && (args.K >= 16384 || wide_env == 2) &&
                    (epi == EPI_F32 || epi == EPI_F32T || epi == EPI_RESID);
  const int bn = (b_mode == B_PAIR) ? GEMM_BN / 2 : (wide ? 2 * GEMM_BN : GEMM_BN);
  args.n_blocks = (args.N + bn - 1) / bn;
  args.k_blocks = (args.K + GEMM_BK - 1) / GEMM_BK;
  // Rasterisation group (pair M-blocks per group): 8 for both schedules
  // (profiles/r01_dyn_group_sweep.log, r01_longk2_group.log; with the dynamic
  // schedule long-K GEMMs preferred 4, with the wave barrier 8).
  static const int g_long = env_int("EE_GEMM_GROUP_LONGK", 8);
  static const int g_short = env_int("EE_GEMM_GROUP_SHORTK", 8);
  if (group > 0)
    args.group_m = group;
  else if (cta_pair)
    args.group_m = args.K >= 16384 ? g_long : g_short;
  else
    args.group_m = 16;
  args.hint_a = hint_a;
  args.hint_b = hint_b;
  args.epi_sleep = epi_sleep;
  args.trace = trace_buffer(args.m_blocks * args.n_blocks);
  if (args.m_blocks == 0 || args.n_blocks == 0 || args.k_blocks == 0) return cudaSuccess;

#define EE_GEMM_CASE(E, AM, BM)                                              \
  if (epi == E && a_mn == AM && b_mn == BM)                                  \
    return cta_pair ? launch2<E, AM, BM>(ta, tb0, tb1, args, st)             \
                    : launch<E, AM, BM>(ta, tb0, tb1, args, st);
#define EE_GEMM_WIDE(E, AM, BM) \
  if (wide && epi == E && a_mn == AM && b_mn == BM) return launch2<E, AM, BM, 2>(ta, tb0, tb1, args, st);
  EE_GEMM_WIDE(EPI_F32, false, false)
  EE_GEMM_WIDE(EPI_F32, false, true)
  EE_GEMM_WIDE(EPI_F32, true, false)
  EE_GEMM_WIDE(EPI_F32, true, true)
  EE_GEMM_WIDE(EPI_F32T, false, true)
  EE_GEMM_WIDE(EPI_RESID, false, false)
#undef EE_GEMM_WIDE
  // the (epilogue, A major, B major) combinations the step uses, plus the
  // plain fp32 GEMM in all four majors (exported for the parity tests)
  EE_GEMM_CASE(EPI_F32, false, false)
  EE_GEMM_CASE(EPI_F32, false, true)
  EE_GEMM_CASE(EPI_F32, true, false)
  EE_GEMM_CASE(EPI_F32, true, true)
  EE_GEMM_CASE(EPI_RESID, false, false)
  EE_GEMM_CASE(EPI_SWIGLU_FWD, false, false)
  EE_GEMM_CASE(EPI_SWIGLU_BWD, false, true)
  EE_GEMM_CASE(EPI_CE_STATS, false, false)
  EE_GEMM_CASE(EPI_CE_DS, false, false)
  EE_GEMM_CASE(EPI_F32T, false, true)
  EE_GEMM_CASE(EPI_F32_ADAM, false, true)
  EE_GEMM_CASE(EPI_F32T_ADAM, false, true)
  EE_GEMM_CASE(EPI_BF16, false, false)
  EE_GEMM_CASE(EPI_BF16, false, true)
#undef EE_GEMM_CASE
  return cudaErrorNotSupported;
}

}  // namespace ee
