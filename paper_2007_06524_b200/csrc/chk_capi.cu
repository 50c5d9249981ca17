// chk_capi.cu -- C ABI (include/chk_pcg.h) over the sm_100a kernels.
//
// Host-side orchestration of the batched PCG (pcg_solve, solver.py:118-194):
// init reductions, one preconditioner apply, then four kernels per iteration;
// convergence is decided on the device, the host only polls an "any realization still
// active" word every few iterations while the next iterations are already queued.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <atomic>
#include <exception>
#include <string>
#include <thread>
#include <type_traits>
#include <vector>

#include "../../include/chk_pcg.h"
#include "chk_kernels.cuh"
#include "chk_sample.cuh"
#include "chk_generic.cuh"

using namespace chk;

namespace {

thread_local std::string g_err;
thread_local long long g_launches = 0;

// Optional per-kernel-class timing with CUDA events on the launching stream
// (the bench's live roofline numbers).  Classes: 0 unused (was a separate
// stencil kernel), 1 fwd_plane, 2 mid_column, 3 inv_plane, 4 other.
struct Profiler {
  bool on = false;
  double ms[5] = {0, 0, 0, 0, 0};
  long long count[5] = {0, 0, 0, 0, 0};
  std::vector<cudaEvent_t> pool;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> open;
  cudaEvent_t take() {
    if (pool.empty()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      return e;
    }
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }
  void collect() {  // call after the stream synchronized
    static FILE* trace = getenv("CHK_PROF_TRACE") ? fopen(getenv("CHK_PROF_TRACE"), "a") : nullptr;
    for (auto& o : open) {
      float t = 0.f;
      if (cudaEventElapsedTime(&t, o.second.first, o.second.second) == cudaSuccess) {
        if (trace) fprintf(trace, "%d %.5f\n", o.first, t);
        ms[o.first] += t;
        count[o.first] += 1;
      }
      pool.push_back(o.second.first);
      pool.push_back(o.second.second);
    }
    open.clear();
    if (trace) fflush(trace);
  }
};
thread_local Profiler g_prof;

struct ProfScope {
  int kind;
  cudaStream_t s;
  cudaEvent_t a = nullptr;
  ProfScope(int k, cudaStream_t st) : kind(k), s(st) {
    if (g_prof.on) {
      a = g_prof.take();
      cudaEventRecord(a, s);
    }
  }
  ~ProfScope() {
    if (a) {
      cudaEvent_t b = g_prof.take();
      cudaEventRecord(b, s);
      g_prof.open.push_back({kind, {a, b}});
    }
  }
};

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CHK_CUDA(call)                                                              \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess) return fail(CHK_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

#define CHK_LAUNCHED()                                                               \
  do {                                                                              \
    ++g_launches;                                                                   \
    cudaError_t e_ = cudaGetLastError();                                            \
    if (e_ != cudaSuccess) return fail(CHK_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(e_)); \
  } while (0)

// Tensor map of the interleaved spectrum layout (n = 256): the exchange buffer as
// a 4-D float64 tensor {4 doubles of a 32-byte piece, G groups (stride 32 B),
// ncols/W pieces (stride G*W*16 B), P*B*nloc rows (stride G*ncols*16 B)}; the
// plane CTAs store / load boxes {4, 1, TmapBox, 1} (cp.async.bulk.tensor).
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

template <int G, int W, int BOX>
static int plane_tmap(const double2* S, int B, const SlabGeo& sg, CUtensorMap* out) {
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return fail(CHK_ECUDA, "cuTensorMapEncodeTiled is not available");
  const cuuint64_t dims[4] = {2 * W, (cuuint64_t)G, (cuuint64_t)(sg.ncols / W), (cuuint64_t)sg.P * B * sg.nloc};
  const cuuint64_t strides[3] = {(cuuint64_t)W * 16, (cuuint64_t)G * W * 16, (cuuint64_t)G * sg.ncols * 16};
  const cuuint32_t box[4] = {2 * W, 1, BOX, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  const CUresult r = enc(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double2*>(S), dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CHK_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return CHK_OK;
}

// Tile geometry per grid size: G interleaved x1 groups per plane slab, W
// spectral columns per middle-pass tile.
template <int N>
struct Cfg;
// NB realizations share one evaluation of the diagonal tile in the middle pass.
#ifndef CHK_W128
#define CHK_W128 8
#endif
// REG: register-resident middle pass (first x0 radix RA in phase A, P
// realizations in flight per CTA); otherwise the shared-memory stage kernel.
template <> struct Cfg<8>   { static constexpr int G = 1,  W = 8,  NB = 4, REG = 1, RA = 8, P = 1; };
template <> struct Cfg<16>  { static constexpr int G = 1,  W = 16, NB = 4, REG = 1, RA = 8, P = 1; };
template <> struct Cfg<32>  { static constexpr int G = 1,  W = 16, NB = 4, REG = 1, RA = 8, P = 1; };
#ifndef CHK_NB64
#define CHK_NB64 4
#endif
#ifndef CHK_NB128
#define CHK_NB128 8  // 16 measured 2.3 % slower in the middle pass (14 long waves; 8 gives 28 shorter ones)
#endif
template <> struct Cfg<64>  { static constexpr int G = 1,  W = 16, NB = CHK_NB64, REG = 1, RA = 8, P = 1; };
template <> struct Cfg<128> { static constexpr int G = 2,  W = CHK_W128, NB = CHK_NB128, REG = 1, RA = 8, P = 1; };
#ifndef CHK_NB256
#define CHK_NB256 8
#endif
template <> struct Cfg<256> { static constexpr int G = 8,  W = 2,  NB = CHK_NB256, REG = 0, RA = 1, P = 1; };
template <> struct Cfg<512> { static constexpr int G = 16, W = 1,  NB = 2, REG = 0, RA = 1, P = 1; };

// every h-cell inside its sub-cell (alpha = 1/2): stencil fast path
// (n0 >= 4, checked by check_grid: every aligned x2 quad lies inside one cell)
inline bool allin(const Geo& g) { return g.k == g.mask + 1 && g.off == 0; }

template <int N>
struct Ops {
  static constexpr int NN = N;
  static constexpr int G = Cfg<N>::G, W = Cfg<N>::W, NB = Cfg<N>::NB, NR = N / G, H = N / 2 + 1;
  static constexpr int REG = Cfg<N>::REG, RA = Cfg<N>::RA, P = Cfg<N>::P;
#ifndef CHK_STAGE
#define CHK_STAGE 1
#endif
  static constexpr bool STG = CHK_STAGE && (N == 64 || N == 128);
  static constexpr int TILES = NR * H / W;
  static constexpr int PLANE_BLOCKS = N * G;  // per realization
  static constexpr size_t plane_smem() { return (size_t)NR * H * sizeof(double2); }
  // shared memory of the fused (n >= 256) middle kernel
  static size_t mid_smem(int r1) {
    return (size_t)mid_dsm_offset(N * (G * W + 1), G * W, r1) + (size_t)N * G * W * sizeof(double);
  }
  // fused middle pass reads the precomputed diagonal from L2 (CHK_MID_DG=0: stage it in smem)
  static bool mid_dg() {
    static const bool on = !(getenv("CHK_MID_DG") && atoi(getenv("CHK_MID_DG")) == 0);
    return on;
  }
  // register middle pass with the residual tile staged by TMA (CHK_MID_RSG=0: off)
  static bool mid_rsg() {
    static const bool on = !(getenv("CHK_MID_RSG") && atoi(getenv("CHK_MID_RSG")) == 0);
    return on;
  }
  static int maxblk() { return PLANE_BLOCKS > TILES ? PLANE_BLOCKS : TILES; }
  // single-GPU layout: all planes, one column chunk, periodic halo inside p
  static SlabGeo whole() { return SlabGeo{N, 0, 1, NR * H, 0, TILES, nullptr, nullptr, 0, N}; }
  // rank `rank` of `P` owning n/P consecutive planes and column chunk `rank`
  static SlabGeo slab(int P, int rank, const double* lo, const double* hi) {
    return SlabGeo{N / P, rank * (N / P), P, NR * H / P, rank * (TILES / P), TILES / P, lo, hi, 0, N / P};
  }
  static bool slab_ok(int P) { return P >= 1 && N % P == 0 && (N / P) >= 1 && TILES % P == 0 && P <= 64; }

  // raise the dynamic shared-memory limit once per (device, kernel instantiation)
  // and size -- the attribute is per device
  template <class K>
  static cudaError_t allow_smem(K kernel, size_t bytes) {
    if (bytes <= 48 * 1024) return cudaSuccess;
    struct Done {
      int dev;
      const void* key;
      size_t bytes;
    };
    static thread_local std::vector<Done> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const void* key = reinterpret_cast<const void*>(kernel);
    for (auto& d : done)
      if (d.dev == dev && d.key == key && d.bytes >= bytes) return cudaSuccess;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) done.push_back({dev, key, bytes});
    return e;
  }

  template <class... KA, class... AA>
  static cudaError_t plaunch(void (*kernel)(KA...), dim3 grid, size_t sm, cudaStream_t s, AA... args) {
    kernel<<<grid, PlaneNT<N>::value, sm, s>>>(args...);
    return cudaSuccess;
  }
  // the interleaved layout's tensor map; *use = 0 (cp.async path) for the contiguous
  // layout or a slab chunk that is not a whole number of boxes
  static int tmap(const double2* S, int B, const SlabGeo& sg, CUtensorMap* tm, int* use) {
    *tm = CUtensorMap{};
    *use = 0;
    if constexpr (IlW<N>::value > 0) {
      if ((sg.ncols / W) % TmapBox<N>::value) return CHK_OK;
      *use = 1;
      return plane_tmap<G, W, TmapBox<N>::value>(S, B, sg, tm);
    }
    return CHK_OK;
  }
  static int fwd(int mode, cudaStream_t s, int B, Geo g, const double* beta, const double* src,
                 double* u, double2* S, PlanDev pl, SolveCtl ctl, int it, SlabGeo sg = whole()) {
    const size_t sm = plane_smem();
    dim3 grid(B * sg.nrun * G);
    CUtensorMap tm;
    int use_tm = 0;
    if (int rc = tmap(S, B, sg, &tm, &use_tm)) return rc;
    ProfScope ps(1, s);
    if (mode == FWD_APPLY) {
      CHK_CUDA(allow_smem(fwd_plane_kernel<N, G, FWD_APPLY, false>, sm));
      CHK_CUDA(plaunch(fwd_plane_kernel<N, G, FWD_APPLY, false>, grid, sm, s, g, beta, src, u, S, pl, ctl, sg, B, it, tm, use_tm));
    } else if (mode == FWD_INIT) {
      CHK_CUDA(allow_smem(fwd_plane_kernel<N, G, FWD_INIT, false>, sm));
      CHK_CUDA(plaunch(fwd_plane_kernel<N, G, FWD_INIT, false>, grid, sm, s, g, beta, src, u, S, pl, ctl, sg, B, it, tm, use_tm));
    } else if (allin(g)) {
      CHK_CUDA(allow_smem(fwd_plane_kernel<N, G, FWD_Q, true>, sm));
      CHK_CUDA(plaunch(fwd_plane_kernel<N, G, FWD_Q, true>, grid, sm, s, g, beta, src, u, S, pl, ctl, sg, B, it, tm, use_tm));
    } else {
      CHK_CUDA(allow_smem(fwd_plane_kernel<N, G, FWD_Q, false>, sm));
      CHK_CUDA(plaunch(fwd_plane_kernel<N, G, FWD_Q, false>, grid, sm, s, g, beta, src, u, S, pl, ctl, sg, B, it, tm, use_tm));
    }
    CHK_LAUNCHED();
    return CHK_OK;
  }
  template <int NBX, int MODE>
  static int mid_launch(cudaStream_t s, int B, double2* S, PlanDev pl, SolveCtl ctl, int it, SlabGeo sg) {
    const int r1 = pl.kind == KIND_LKR ? pl.r1 : 0;
    dim3 grid(((B + NBX - 1) / NBX) * sg.tiles), block(MidNT<N>::value);
    if constexpr (REG) {
      constexpr int PX = (NBX == 1) ? 1 : P;
      constexpr int NT = (W * (N / RA) > 128 ? 256 : 128) * PX;
      constexpr bool SX = STG && PX == 1 && W * (N / RA) == NT;
      // staged residual + diagonal in registers: n = 128 only (mid -1.7 % time; n = 64 +2 %)
      constexpr bool RX = SX && (G * W * RA == NT) && N == 128;
      if (RX && pl.D && mid_rsg()) {
        const size_t sm = (((size_t)N * (G * W + 1) * sizeof(double2) + 127) & ~(size_t)127) +
                          (size_t)N * G * W * sizeof(double2) + (size_t)G * RA * NT * sizeof(double2);
        CHK_CUDA(allow_smem(mid_column_reg_kernel<N, G, W, RA, NBX, PX, MODE, NT, SX, RX>, sm));
        mid_column_reg_kernel<N, G, W, RA, NBX, PX, MODE, NT, SX, RX><<<grid, NT, sm, s>>>(S, pl, ctl, sg, it, B);
        return CHK_OK;
      }
      size_t sm = (size_t)mid_dsm_offset(PX * N * (G * W + 1), G * W, r1) + (((size_t)N * G * W * sizeof(double) + 15) & ~(size_t)15);
      if (SX) sm += (size_t)G * RA * NT * sizeof(double2);
      CHK_CUDA(allow_smem(mid_column_reg_kernel<N, G, W, RA, NBX, PX, MODE, NT, SX>, sm));
      mid_column_reg_kernel<N, G, W, RA, NBX, PX, MODE, NT, SX><<<grid, NT, sm, s>>>(S, pl, ctl, sg, it, B);
    } else if (N == 256 && CHK_R256) {
      // register-phase kernel (x0 radix order 2, 8, 8, 2; diagonal from the plan table)
      if (!pl.D) return fail(CHK_EINVAL, "n = 256 middle pass needs the plan's diagonal table");
      const size_t sm = (size_t)N * CHK_R256_RS * sizeof(double2);
      CHK_CUDA(allow_smem(mid_column_r256_kernel<NBX, MODE>, sm));
      mid_column_r256_kernel<NBX, MODE><<<grid, 256, sm, s>>>(S, pl, ctl, sg, it, B);
    } else if (pl.D && mid_dg()) {
      const size_t sm = (size_t)N * (G * W + 1) * sizeof(double2);
      CHK_CUDA(allow_smem(mid_column_fused_kernel<N, G, W, NBX, MODE, true>, sm));
      mid_column_fused_kernel<N, G, W, NBX, MODE, true><<<grid, block, sm, s>>>(S, pl, ctl, sg, it, B);
    } else {
      const size_t sm = mid_smem(r1);
      CHK_CUDA(allow_smem(mid_column_fused_kernel<N, G, W, NBX, MODE>, sm));
      mid_column_fused_kernel<N, G, W, NBX, MODE><<<grid, block, sm, s>>>(S, pl, ctl, sg, it, B);
    }
    return CHK_OK;
  }
  static int mid(int mode, cudaStream_t s, int B, double2* S, PlanDev pl, SolveCtl ctl, int it,
                 SlabGeo sg = whole()) {
    ProfScope ps(2, s);
    // amortise the diagonal over NB realizations per CTA when that still gives
    // >= 2 CTAs per SM (measured: the diagonal tile costs more than wave fill)
    const int pick = ((long long)((B + NB - 1) / NB) * sg.tiles >= 2LL * 148) ? NB : 1;
    int rc;
    auto go = [&](auto mode_tag) -> int {
      constexpr int M = decltype(mode_tag)::value;
      if (pick == NB) return mid_launch<NB, M>(s, B, S, pl, ctl, it, sg);
      if (pick == 4) return mid_launch<(NB > 4 ? 4 : NB), M>(s, B, S, pl, ctl, it, sg);
      return mid_launch<1, M>(s, B, S, pl, ctl, it, sg);
    };
    if (mode == MID_APPLY)
      rc = go(std::integral_constant<int, MID_APPLY>{});
    else if (mode == MID_INIT)
      rc = go(std::integral_constant<int, MID_INIT>{});
    else
      rc = go(std::integral_constant<int, MID_ITER>{});
    if (rc) return rc;
    CHK_LAUNCHED();
    return CHK_OK;
  }
  static int inv(int mode, cudaStream_t s, int B, const double2* S, double* out, double* u,
                 PlanDev pl, SolveCtl ctl, int it, SlabGeo sg = whole()) {
    const size_t sm = plane_smem();
    dim3 grid(B * sg.nrun * G);
    CUtensorMap tm;
    int use_tm = 0;
    if (int rc = tmap(S, B, sg, &tm, &use_tm)) return rc;
    ProfScope ps(3, s);
    if (mode == INV_APPLY) {
      CHK_CUDA(allow_smem(inv_plane_kernel<N, G, INV_APPLY>, sm));
      CHK_CUDA(plaunch(inv_plane_kernel<N, G, INV_APPLY>, grid, sm, s, S, out, u, pl, ctl, sg, B, it, tm, use_tm));
    } else if (mode == INV_INIT) {
      CHK_CUDA(allow_smem(inv_plane_kernel<N, G, INV_INIT>, sm));
      CHK_CUDA(plaunch(inv_plane_kernel<N, G, INV_INIT>, grid, sm, s, S, out, u, pl, ctl, sg, B, it, tm, use_tm));
    } else {
      CHK_CUDA(allow_smem(inv_plane_kernel<N, G, INV_ITER>, sm));
      CHK_CUDA(plaunch(inv_plane_kernel<N, G, INV_ITER>, grid, sm, s, S, out, u, pl, ctl, sg, B, it, tm, use_tm));
    }
    CHK_LAUNCHED();
    return CHK_OK;
  }
  // paired plane pass (pair_plane_kernel): fa.blocks forward + ia.blocks inverse CTAs
  static int pair(cudaStream_t s, const FwdArgs& fa, const InvArgs& ia, PlanDev pl) {
    const size_t sm = plane_smem();
    const SlabGeo sg = whole();
    dim3 grid(fa.blocks + ia.blocks), block(PlaneNT<N>::value);
    ProfScope ps(4, s);
    if (allin(fa.g)) {
      CHK_CUDA(allow_smem(pair_plane_kernel<N, G, true>, sm));
      pair_plane_kernel<N, G, true><<<grid, block, sm, s>>>(fa, ia, pl, sg);
    } else {
      CHK_CUDA(allow_smem(pair_plane_kernel<N, G, false>, sm));
      pair_plane_kernel<N, G, false><<<grid, block, sm, s>>>(fa, ia, pl, sg);
    }
    CHK_LAUNCHED();
    return CHK_OK;
  }
  static int stencil(cudaStream_t s, int B, Geo g, const double* beta, const double* x, double* y,
                     double* xy, double* part, unsigned* cnt) {
    if (allin(g))
      stencil_apply_kernel<N, G, true><<<B * PLANE_BLOCKS, 256, 0, s>>>(g, beta, x, y, xy, part, cnt);
    else
      stencil_apply_kernel<N, G, false><<<B * PLANE_BLOCKS, 256, 0, s>>>(g, beta, x, y, xy, part, cnt);
    CHK_LAUNCHED();
    return CHK_OK;
  }
  static int rhs_stats(cudaStream_t s, int B, const double* f, SolveCtl ctl, SlabGeo sg = whole()) {
    rhs_stats_kernel<N, G><<<B * sg.nloc * G, 256, 0, s>>>(f, ctl, sg);
    CHK_LAUNCHED();
    return CHK_OK;
  }
  static int mean_u(cudaStream_t s, int B, const double* u, SolveCtl ctl, SlabGeo sg = whole()) {
    mean_u_kernel<N, G><<<B * sg.nloc * G, 256, 0, s>>>(u, ctl, sg);
    CHK_LAUNCHED();
    return CHK_OK;
  }
  static int rhs(cudaStream_t s, int B, Geo g, const double* beta, double* f, int axis, double scale) {
    dim3 grid(296, B);
    corrector_rhs_kernel<N><<<grid, 256, 0, s>>>(g, beta, f, axis, scale);
    CHK_LAUNCHED();
    return CHK_OK;
  }
};

#define CHK_DISPATCH(n, ...)                               \
  switch (n) {                                             \
    case 8:   { using O = Ops<8>;   __VA_ARGS__; } break;  \
    case 16:  { using O = Ops<16>;  __VA_ARGS__; } break;  \
    case 32:  { using O = Ops<32>;  __VA_ARGS__; } break;  \
    case 64:  { using O = Ops<64>;  __VA_ARGS__; } break;  \
    case 128: { using O = Ops<128>; __VA_ARGS__; } break;  \
    case 256: { using O = Ops<256>; __VA_ARGS__; } break;  \
    case 512: { using O = Ops<512>; __VA_ARGS__; } break;  \
    default: return fail(CHK_EUNSUPPORTED, "unsupported n " + std::to_string(n)); \
  }

// CHK_DISPATCH for contexts that cannot return (sets rc on an unsupported n)
#define CHK_DISPATCH_V(n, rc, ...)                         \
  switch (n) {                                             \
    case 8:   { using O = Ops<8>;   __VA_ARGS__; } break;  \
    case 16:  { using O = Ops<16>;  __VA_ARGS__; } break;  \
    case 32:  { using O = Ops<32>;  __VA_ARGS__; } break;  \
    case 64:  { using O = Ops<64>;  __VA_ARGS__; } break;  \
    case 128: { using O = Ops<128>; __VA_ARGS__; } break;  \
    case 256: { using O = Ops<256>; __VA_ARGS__; } break;  \
    case 512: { using O = Ops<512>; __VA_ARGS__; } break;  \
    default: rc = fail(CHK_EUNSUPPORTED, "unsupported n"); \
  }

// Realizations in the first half of a paired solve (0: unpaired).  Pairing pays
// at n = 128 only, while each half alone still fills >= 2 CTAs per SM in the
// middle pass (measured: config 3 +1.4 %; config 2 (n = 64) -19 %, config 4
// (n = 256) -1.5 %).  CHK_PAIR=0 disables it, CHK_PAIR=2 forces it for any
// B >= 2 (tests).
template <class O>
int pair_split(int B) {
  const char* e = getenv("CHK_PAIR");
  const int env = e ? atoi(e) : 1;
  if (env == 2 && B >= 2) return B / 2;
  if (!env || !O::REG || O::NN != 128 || B < 2 * O::NB) return 0;
  const int Ba = (B / 2) / O::NB * O::NB;
  const int Bb = B - Ba;
  const long long ctas = (long long)(Ba / O::NB) * O::TILES;
  return (ctas >= 2LL * 148 && Bb >= Ba) ? Ba : 0;
}

// fused fast path: the power-of-two sizes of the BASELINE configurations
bool supported_n(int n) { return n >= 8 && n <= 512 && (n & (n - 1)) == 0; }
// every other n = n0 * L (n0 a power of two >= 4, so n is a multiple of 4) runs the
// generic kernels (chk_generic.cuh); the direct Fourier sums stage 16 lines of n
// complex values in shared memory, which bounds n
constexpr int GEN_MAX_N = 720;
constexpr int GEN_TL = 16;
bool generic_n(int n) { return n >= 4 && n <= GEN_MAX_N && n % 4 == 0 && !supported_n(n); }
bool any_n(int n) { return supported_n(n) || generic_n(n); }

int maxblk_of(int n) {
  int m = 0;
  if (generic_n(n)) return n;
  switch (n) {
    case 8: m = Ops<8>::maxblk(); break;
    case 16: m = Ops<16>::maxblk(); break;
    case 32: m = Ops<32>::maxblk(); break;
    case 64: m = Ops<64>::maxblk(); break;
    case 128: m = Ops<128>::maxblk(); break;
    case 256: m = Ops<256>::maxblk(); break;
    case 512: m = Ops<512>::maxblk(); break;
  }
  return m;
}

int check_grid(const chk_grid* g, Geo* out) {
  if (!g) return fail(CHK_EINVAL, "grid is NULL");
  if (g->d != 3) return fail(CHK_EUNSUPPORTED, "only d = 3 is implemented on the GPU path");
  if (!any_n(g->n))
    return fail(CHK_EUNSUPPORTED, "n must be a multiple of 4 in [4, " + std::to_string(GEN_MAX_N) + "] (or a power of two <= 512)");
  if (g->n0 < 4 || (g->n0 & (g->n0 - 1)) || g->L < 1 || g->n0 * g->L != g->n)  // lattice.py:122-123
    return fail(CHK_EINVAL, "need n = n0 * L with n0 a power of two >= 4");
  if (g->k < 1 || g->k > g->n0 || g->offset < 0 || g->offset + g->k > g->n0)
    return fail(CHK_EINVAL, "sub-cell window outside the cell");
  if (!(g->lam > 0.0)) return fail(CHK_EINVAL, "lambda must be positive");
  int sh = 0;
  while ((1 << sh) < g->n0) ++sh;
  *out = Geo{g->n, g->L, sh, g->n0 - 1, g->k, g->offset, g->lam};
  return CHK_OK;
}

size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

struct Workspace {
  double* p;
  double2* Rh;
  double2* S;
  double* part;
  RState* st;
  double* hist;
  size_t bytes;
  // generic sizes: residual and q / z in real space, rank-free reduction slots
  double* r;
  double* q;
  double* red;
};

Workspace carve(void* base, int n, int B, int max_iter) {
  const size_t nb = (size_t)n * n * n;
  const size_t spec = (size_t)n * n * (n / 2 + 1);
  char* c = static_cast<char*>(base);
  Workspace w{};
  size_t off = 0;
  if (generic_n(n)) {
    w.p = reinterpret_cast<double*>(c + off); off = align_up(off + sizeof(double) * nb * B);
    w.r = reinterpret_cast<double*>(c + off); off = align_up(off + sizeof(double) * nb * B);
    w.q = reinterpret_cast<double*>(c + off); off = align_up(off + sizeof(double) * nb * B);
    w.S = reinterpret_cast<double2*>(c + off); off = align_up(off + sizeof(double2) * nb * B);
    w.part = reinterpret_cast<double*>(c + off); off = align_up(off + sizeof(double) * 2 * (size_t)n * B);
    w.red = reinterpret_cast<double*>(c + off); off = align_up(off + sizeof(double) * 4 * (size_t)B);
    w.st = reinterpret_cast<RState*>(c + off); off = align_up(off + sizeof(RState) * B);
    w.hist = reinterpret_cast<double*>(c + off); off = align_up(off + sizeof(double) * (size_t)max_iter * B);
    w.bytes = off;
    return w;
  }
  w.p = reinterpret_cast<double*>(c + off); off = align_up(off + sizeof(double) * nb * B);
  w.Rh = reinterpret_cast<double2*>(c + off); off = align_up(off + sizeof(double2) * spec * B);
  w.S = reinterpret_cast<double2*>(c + off); off = align_up(off + sizeof(double2) * spec * B);
  w.part = reinterpret_cast<double*>(c + off); off = align_up(off + sizeof(double) * 2 * (size_t)maxblk_of(n) * B);
  w.st = reinterpret_cast<RState*>(c + off); off = align_up(off + sizeof(RState) * B);
  w.hist = reinterpret_cast<double*>(c + off); off = align_up(off + sizeof(double) * (size_t)max_iter * B);
  w.bytes = off;
  return w;
}

struct PinnedStates {
  RState* h = nullptr;
  size_t cap = 0;
  int* flags = nullptr;  // [2] "any realization still active" words written by poll_active_kernel
  ~PinnedStates() {
    if (h) cudaFreeHost(h);
    if (flags) cudaFreeHost(flags);
    if (hist) cudaFreeHost(hist);
  }
  // Host-mapped words for the convergence poll.  The device writes them itself (zero-copy
  // store from a one-CTA kernel) instead of a cudaMemcpyAsync: a status copy queues on the
  // device-to-host copy engine behind any bulk download in flight (another pipeline lane's
  // 0.5 GB of solutions, ~10 ms), the polling host thread then waits that long, and with
  // only a few iterations of look-ahead queued the GPU ran dry (a 4 GiB download beside a
  // config-3 solve cost 50 ms this way).
  int* poll_flags() {
    if (!flags && cudaHostAlloc(&flags, 64, cudaHostAllocMapped) != cudaSuccess) flags = nullptr;
    return flags;
  }
  // pinned staging of the residual histories (same reason: written by the device itself)
  double* hist = nullptr;
  size_t hist_cap = 0;
  double* get_hist(size_t n) {
    if (n > hist_cap) {
      if (hist) cudaFreeHost(hist);
      hist = nullptr;
      hist_cap = 0;
      if (cudaMallocHost(&hist, n * sizeof(double)) != cudaSuccess) return hist = nullptr;
      hist_cap = n;
    }
    return hist;
  }
  RState* get(size_t n) {
    if (n > cap) {
      if (h) cudaFreeHost(h);
      h = nullptr;
      if (cudaMallocHost(&h, n * sizeof(RState)) != cudaSuccess) {
        h = nullptr;
        cap = 0;
        return nullptr;
      }
      cap = n;
    }
    return h;
  }
};
thread_local PinnedStates g_pinned;

// n 8-byte words device -> pinned host memory by zero-copy stores (small read-backs that must
// not queue behind bulk downloads on the copy engine)
__global__ void words_to_host_kernel(const unsigned long long* __restrict__ src, unsigned long long* dst, size_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
  __threadfence_system();
}

// out[0] = 1 while any realization is still active (host-mapped memory, see poll_flags)
__global__ void poll_active_kernel(const RState* __restrict__ st, int B, int* out) {
  __shared__ int any;
  if (threadIdx.x == 0) any = 0;
  __syncthreads();
  int a = 0;
  for (int b = threadIdx.x; b < B; b += blockDim.x) a |= (st[b].status == ST_ACTIVE);
  if (a) any = 1;
  __syncthreads();
  if (threadIdx.x == 0) {
    *out = any;
    __threadfence_system();
  }
}

// Per-realization states (and optionally the residual histories) back to the host after a
// solve: zero-copy kernels into pinned memory, one stream synchronize, then plain host copies.
static_assert(sizeof(RState) % 8 == 0, "RState is copied as 8-byte words");
int read_back(const Workspace& w, int B, int max_iter, int32_t* iterations, double* final_rel, int32_t* status,
              int32_t* rhs_projected, double* history, cudaStream_t s) {
  RState* hst = g_pinned.get((size_t)B);
  if (!hst) return fail(CHK_ECUDA, "cudaMallocHost failed");
  words_to_host_kernel<<<4, 256, 0, s>>>(reinterpret_cast<const unsigned long long*>(w.st),
                                        reinterpret_cast<unsigned long long*>(hst), sizeof(RState) / 8 * (size_t)B);
  CHK_LAUNCHED();
  double* hh = nullptr;
  const size_t nh = (size_t)max_iter * B;
  if (history) {
    hh = g_pinned.get_hist(nh);
    if (!hh) return fail(CHK_ECUDA, "cudaMallocHost failed");
    words_to_host_kernel<<<32, 256, 0, s>>>(reinterpret_cast<const unsigned long long*>(w.hist),
                                           reinterpret_cast<unsigned long long*>(hh), nh);
    CHK_LAUNCHED();
  }
  CHK_CUDA(cudaStreamSynchronize(s));
  if (history) memcpy(history, hh, sizeof(double) * nh);
  for (int b = 0; b < B; ++b) {
    int stt = hst[b].status;
    if (stt == ST_ACTIVE) stt = ST_NOT_CONVERGED;  // defensive; max_iter always decides
    if (status) status[b] = stt;
    if (iterations) iterations[b] = hst[b].iters;
    if (final_rel) final_rel[b] = hst[b].final_rel;
    if (rhs_projected) rhs_projected[b] = hst[b].rhs_projected;
  }
  return CHK_OK;
}

// ---- generic grid sizes (chk_generic.cuh) ----
// z = P x for the B complex arrays already in S (x + 0 i): forward sums along x2,
// x1, x0, scaling by D / n^3, inverse sums along x0, x1, x2 (the last one leaves
// the real part in z).  st != null: only active realizations.
int gen_precond(cudaStream_t s, int B, int n, double2* S, const PlanDev& pl, int project, const RState* st,
                double* z) {
  const size_t sm = sizeof(double2) * ((size_t)n * GEN_TL + n);
  CHK_CUDA(Ops<8>::allow_smem(gen_dft_axis_kernel<false>, sm));
  CHK_CUDA(Ops<8>::allow_smem(gen_dft_axis_kernel<true>, sm));
  const dim3 grid((n * n + GEN_TL - 1) / GEN_TL, B);
  for (int axis = 2; axis >= 0; --axis) {
    gen_dft_axis_kernel<false><<<grid, 256, sm, s>>>(S, pl.tw, n, axis, GEN_TL, st, nullptr);
    CHK_LAUNCHED();
  }
  gen_scale_kernel<<<dim3(n, B), 256, 0, s>>>(S, pl, n, project, st);
  CHK_LAUNCHED();
  for (int axis = 0; axis <= 2; ++axis) {
    gen_dft_axis_kernel<true><<<grid, 256, sm, s>>>(S, pl.tw, n, axis, GEN_TL, st, axis == 2 ? z : nullptr);
    CHK_LAUNCHED();
  }
  return CHK_OK;
}

// Batched PCG (solver.py:118-194) for a generic grid size; same per-realization
// state, decisions (decide_kernel) and reporting as the fused path.
int gen_solve(const Geo& g, const PlanDev& pl, const double* beta, const double* f, double* u, int B,
              const chk_pcg_opts* opts, int32_t* iterations, double* final_rel, int32_t* status,
              int32_t* rhs_projected, double* history, const Workspace& w, cudaStream_t s) {
  const int n = g.n;
  const double ntot = (double)n * n * n;
  const dim3 grid(n, B);
  SolveCtl ctl{w.st, nullptr, w.part, w.hist, n, opts->max_iter, opts->tol, opts->precond_residual_stopping ? 1 : 0,
               w.red, 0};
  int* flags = g_pinned.poll_flags();
  if (!flags) return fail(CHK_ECUDA, "cudaMallocHost failed");
  CHK_CUDA(cudaMemsetAsync(w.st, 0, sizeof(RState) * B, s));
  CHK_CUDA(cudaMemsetAsync(w.hist, 0, sizeof(double) * (size_t)opts->max_iter * B, s));
  CHK_CUDA(cudaMemsetAsync(w.red, 0, sizeof(double) * 4 * B, s));
  cudaEvent_t ev[2];
  CHK_CUDA(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
  CHK_CUDA(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
  auto finalize = [&](int slot0, int slot1) -> int {
    gen_finalize_kernel<<<B, 256, 0, s>>>(w.part, n, slot0 >= 0 ? w.red + slot0 : nullptr,
                                          slot1 >= 0 ? w.red + slot1 : nullptr, 4);
    CHK_LAUNCHED();
    return CHK_OK;
  };
  auto decide = [&](int what, int it) -> int {
    decide_kernel<<<1, 256, 0, s>>>(ctl, w.red, B, what, it, ntot);
    CHK_LAUNCHED();
    return CHK_OK;
  };
  // z = P r (mean-projected) into w.q, then ||r||^2 and r.z, decisions, direction update
  auto precond_step = [&](int it) -> int {
    int rc2;
    gen_residual_kernel<<<grid, 256, 0, s>>>(w.r, w.q, w.S, n, w.st, it);
    CHK_LAUNCHED();
    if ((rc2 = gen_precond(s, B, n, w.S, pl, 1, w.st, w.q))) return rc2;
    gen_dots_kernel<<<grid, 256, 0, s>>>(w.r, w.q, n, w.part, w.st);
    CHK_LAUNCHED();
    if ((rc2 = finalize(1, 2))) return rc2;
    if ((rc2 = decide(DECIDE_MID, it))) return rc2;
    gen_update_kernel<<<grid, 256, 0, s>>>(w.p, u, w.q, n, w.st, it);
    CHK_LAUNCHED();
    return CHK_OK;
  };
  auto run = [&]() -> int {
    int rc2;
    // r = f (projected), u = 0, z = P r, p = z  (solver.py:131-156)
    gen_stats_kernel<<<grid, 256, 0, s>>>(f, n, w.part);
    CHK_LAUNCHED();
    if ((rc2 = finalize(0, 1))) return rc2;
    if ((rc2 = decide(DECIDE_STATS, 0))) return rc2;
    gen_init_kernel<<<grid, 256, 0, s>>>(f, w.r, u, n, w.st);
    CHK_LAUNCHED();
    if ((rc2 = precond_step(0))) return rc2;
    const int chunk = 4;
    bool pending = false;
    int ev_i = 0;
    for (int it = 1; it <= opts->max_iter; ++it) {
      // q = A p, p.q -> alpha (solver.py:162-166)
      gen_stencil_kernel<<<grid, 256, 0, s>>>(g, beta, w.p, w.q, w.part, w.st);
      CHK_LAUNCHED();
      if ((rc2 = finalize(0, -1))) return rc2;
      if ((rc2 = decide(DECIDE_ALPHA, it))) return rc2;
      // r -= alpha q, stop test, z = P r, beta, u += alpha p, p = z + beta p (solver.py:167-184)
      if ((rc2 = precond_step(it))) return rc2;
      if (it % chunk == 0 || it == opts->max_iter) {
        if (pending) {
          CHK_CUDA(cudaEventSynchronize(ev[ev_i ^ 1]));
          if (!reinterpret_cast<volatile int*>(flags)[ev_i ^ 1]) break;
        }
        poll_active_kernel<<<1, 256, 0, s>>>(w.st, B, flags + ev_i);
        CHK_LAUNCHED();
        CHK_CUDA(cudaEventRecord(ev[ev_i], s));
        ev_i ^= 1;
        pending = true;
      }
    }
    // final projection of u (solver.py:169; applied once)
    gen_sum_kernel<<<grid, 256, 0, s>>>(u, n, w.part);
    CHK_LAUNCHED();
    if ((rc2 = finalize(3, -1))) return rc2;
    if ((rc2 = decide(DECIDE_MEANU, 0))) return rc2;
    sub_mean_kernel<<<1184, 256, 0, s>>>(u, w.st, (size_t)n * n * n, B);
    CHK_LAUNCHED();
    return CHK_OK;
  };
  const int rc = run();
  cudaEventDestroy(ev[0]);
  cudaEventDestroy(ev[1]);
  if (rc) return rc;
  return read_back(w, B, opts->max_iter, iterations, final_rel, status, rhs_projected, history, s);
}

}  // namespace

struct chk_precond_plan {
  int kind;
  int n;
  int r1;
  double delta;
  double2* d_tw;
  double* d_U;
  double* d_Up;
  double* d_lam;
  double* d_D;  // [tiles][n][G*W] diagonal tiles, computed once at plan creation
};

static PlanDev plan_dev(const chk_precond_plan* p) {
  return PlanDev{p->d_tw, p->d_U, p->d_Up, p->d_lam, p->r1, p->kind, p->delta, p->d_D};
}

// host copy of dig_freq0 (chk_kernels.cuh): frequency stored at x0 position p
static int host_dig_freq(int N, int p) {
  int k = 0, mul = 1, M = N;
  while (M > 1) {
    const int R = x0_radix(N, M);
    const int Mn = M / R;
    const int m = p / Mn;
    p -= m * Mn;
    k += m * mul;
    mul *= R;
    M = Mn;
  }
  return k;
}

// Evaluate every diagonal tile of a plan into p->d_D (dtile_kernel).
static int plan_dtiles(chk_precond_plan* p) {
  const int n = p->n;
  const size_t nd = (size_t)n * n * (n / 2 + 1);
  CHK_CUDA(cudaMalloc(&p->d_D, sizeof(double) * nd));
  PlanDev pl = plan_dev(p);
  pl.D = nullptr;
  CHK_DISPATCH(n, {
    constexpr int GW = O::G * O::W;
    const size_t sm = sizeof(double) * (((size_t)p->r1 * GW + 1) / 2 * 2 + (size_t)n * GW);
    CHK_CUDA(O::allow_smem(dtile_kernel<O::NN, O::G, O::W>, sm));
    dtile_kernel<O::NN, O::G, O::W><<<O::TILES, 256, sm>>>(pl, p->d_D);
    CHK_LAUNCHED();
  });
  CHK_CUDA(cudaDeviceSynchronize());
  return CHK_OK;
}

extern "C" {

int32_t chk_abi_version(void) { return 1; }
const char* chk_last_error(void) { return g_err.c_str(); }
int64_t chk_last_launch_count(void) { return g_launches; }

int32_t chk_profile_enable(int32_t on) {
  g_prof.collect();
  g_prof.on = on != 0;
  for (int i = 0; i < 5; ++i) {
    g_prof.ms[i] = 0.0;
    g_prof.count[i] = 0;
  }
  return CHK_OK;
}

int32_t chk_profile_read(double* ms, int64_t* launches) {
  g_prof.collect();
  for (int i = 0; i < 5; ++i) {
    if (ms) ms[i] = g_prof.ms[i];
    if (launches) launches[i] = g_prof.count[i];
  }
  return CHK_OK;
}

int32_t chk_precond_plan_create(int32_t kind, int32_t n, int32_t r1, const double* factors,
                                const double* eigenvalues, double delta, chk_precond_plan** out) {
  if (!out) return fail(CHK_EINVAL, "out is NULL");
  *out = nullptr;
  if (!any_n(n)) return fail(CHK_EUNSUPPORTED, "unsupported grid size n = " + std::to_string(n));
  if (kind != CHK_PRECOND_LKR && kind != CHK_PRECOND_FOURIER && kind != CHK_PRECOND_REGULARIZED)
    return fail(CHK_EINVAL, "unknown preconditioner kind");
  if (kind == CHK_PRECOND_LKR && (factors == nullptr || r1 < 1 || r1 > 512))
    return fail(CHK_EINVAL, "LKR plan needs factors [3][r1][n] with 1 <= r1 <= 512");
  if (kind != CHK_PRECOND_LKR && eigenvalues == nullptr)
    return fail(CHK_EINVAL, "Fourier plans need the eigenvalues");
  if (kind == CHK_PRECOND_REGULARIZED && delta < 0.0) return fail(CHK_EINVAL, "delta must be >= 0");
  auto* p = new chk_precond_plan{kind, n, kind == CHK_PRECOND_LKR ? r1 : 0, delta, nullptr, nullptr, nullptr, nullptr,
                                 nullptr};
  // twiddles w[k] = exp(-2 pi i k / n), octant-reduced for symmetric accuracy
  std::vector<double2> tw(n);
  for (int k = 0; k < n; ++k) {
    // angle = 2 pi k / n; use the exactly representable fraction k/n
    long double a = 2.0L * 3.14159265358979323846264338327950288L * (long double)k / (long double)n;
    tw[k] = make_double2((double)cosl(a), (double)(-sinl(a)));
  }
  // exact values at the quadrant points
  tw[0] = make_double2(1.0, 0.0);
  if (n % 4 == 0) {
    tw[n / 4] = make_double2(0.0, -1.0);
    tw[n / 2] = make_double2(-1.0, 0.0);
    tw[3 * n / 4] = make_double2(0.0, 1.0);
  }
  cudaError_t e;
  {
    // constant-memory twiddles of the plane passes (c_tw512; per device, same values every time)
    std::vector<double2> t5(512);
    for (int k = 0; k < 512; ++k) {
      long double a = 2.0L * 3.14159265358979323846264338327950288L * (long double)k / 512.0L;
      t5[k] = make_double2((double)cosl(a), (double)(-sinl(a)));
    }
    t5[0] = make_double2(1.0, 0.0);
    t5[128] = make_double2(0.0, -1.0);
    t5[256] = make_double2(-1.0, 0.0);
    t5[384] = make_double2(0.0, 1.0);
    if ((e = cudaMemcpyToSymbol(c_tw512, t5.data(), sizeof(double2) * 512)) != cudaSuccess) goto cuda_fail;
  }
  if ((e = cudaMalloc(&p->d_tw, sizeof(double2) * n)) != cudaSuccess) goto cuda_fail;
  if ((e = cudaMemcpy(p->d_tw, tw.data(), sizeof(double2) * n, cudaMemcpyHostToDevice)) != cudaSuccess) goto cuda_fail;
  if (kind == CHK_PRECOND_LKR) {
    if ((e = cudaMalloc(&p->d_U, sizeof(double) * 3 * (size_t)r1 * n)) != cudaSuccess) goto cuda_fail;
    if ((e = cudaMemcpy(p->d_U, factors, sizeof(double) * 3 * (size_t)r1 * n, cudaMemcpyHostToDevice)) != cudaSuccess) goto cuda_fail;
    if (supported_n(n)) {
      std::vector<double> up((size_t)r1 * n);
      for (int r = 0; r < r1; ++r)
        for (int q = 0; q < n; ++q) up[(size_t)r * n + q] = factors[(size_t)r * n + host_dig_freq(n, q)];
      if ((e = cudaMalloc(&p->d_Up, sizeof(double) * up.size())) != cudaSuccess) goto cuda_fail;
      if ((e = cudaMemcpy(p->d_Up, up.data(), sizeof(double) * up.size(), cudaMemcpyHostToDevice)) != cudaSuccess) goto cuda_fail;
    }
  } else {
    if ((e = cudaMalloc(&p->d_lam, sizeof(double) * n)) != cudaSuccess) goto cuda_fail;
    if ((e = cudaMemcpy(p->d_lam, eigenvalues, sizeof(double) * n, cudaMemcpyHostToDevice)) != cudaSuccess) goto cuda_fail;
  }
  // diagonal tiles of every middle-pass tile (n^2 (n/2+1) doubles: 8.5 MB at
  // n = 128, 539 MB at n = 512); CHK_NO_DTILE=1 evaluates them per CTA instead
  // (n = 256 always has the table: its middle pass reads it)
  if (supported_n(n) && (!(getenv("CHK_NO_DTILE") && atoi(getenv("CHK_NO_DTILE"))) || (n == 256 && CHK_R256))) {
    const int rc2 = plan_dtiles(p);
    if (rc2) {
      chk_precond_plan_destroy(p);
      return rc2;
    }
  }
  *out = p;
  return CHK_OK;
cuda_fail:
  chk_precond_plan_destroy(p);
  return fail(CHK_ECUDA, std::string("plan create: ") + cudaGetErrorString(e));
}

int32_t chk_precond_plan_destroy(chk_precond_plan* p) {
  if (!p) return CHK_OK;
  if (p->d_tw) cudaFree(p->d_tw);
  if (p->d_U) cudaFree(p->d_U);
  if (p->d_Up) cudaFree(p->d_Up);
  if (p->d_lam) cudaFree(p->d_lam);
  if (p->d_D) cudaFree(p->d_D);
  delete p;
  return CHK_OK;
}

size_t chk_precond_workspace_bytes(const chk_precond_plan* p, int32_t B) {
  if (!p || B < 1) return 0;
  const size_t n = p->n;
  if (generic_n(p->n)) return align_up(sizeof(double2) * n * n * n * (size_t)B);
  return align_up(sizeof(double2) * n * n * (n / 2 + 1) * (size_t)B);
}

int32_t chk_precond_apply(const chk_precond_plan* p, const double* r, double* z, int32_t B,
                          void* workspace, size_t workspace_bytes, void* stream) {
  if (!p || !r || !z || B < 1) return fail(CHK_EINVAL, "bad arguments");
  if (!workspace || workspace_bytes < chk_precond_workspace_bytes(p, B))
    return fail(CHK_EINVAL, "workspace too small");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  double2* S = static_cast<double2*>(workspace);
  PlanDev pl = plan_dev(p);
  SolveCtl ctl{};
  Geo g{};
  g.n = p->n;
  int rc = CHK_OK;
  if (generic_n(p->n)) {
    gen_load_kernel<<<dim3(p->n, B), 256, 0, s>>>(r, S, p->n);
    CHK_LAUNCHED();
    return gen_precond(s, B, p->n, S, pl, 0, nullptr, z);
  }
  CHK_DISPATCH(p->n, {
    rc = O::fwd(FWD_APPLY, s, B, g, nullptr, r, nullptr, S, pl, ctl, 0);
    if (rc) return rc;
    rc = O::mid(MID_APPLY, s, B, S, pl, ctl, 0);
    if (rc) return rc;
    rc = O::inv(INV_APPLY, s, B, S, z, nullptr, pl, ctl, 0);
  });
  return rc;
}

int32_t chk_stencil_apply(const chk_grid* grid, const double* beta, const double* x, double* y,
                          double* xy, int32_t B, void* stream) {
  Geo g;
  int rc = check_grid(grid, &g);
  if (rc) return rc;
  if (!beta || !x || !y || B < 1) return fail(CHK_EINVAL, "bad arguments");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  double* part = nullptr;
  unsigned* cnt = nullptr;
  if (xy) {
    // per-CTA partials + tickets of <x, y>: a scratch buffer per (thread, device,
    // stream) kept across calls (grown on demand; the tickets are zeroed in stream
    // order every call), so overlapping calls on different streams never share it
    struct Scratch {
      int dev = -1;
      cudaStream_t stream = nullptr;
      void* p = nullptr;
      size_t cap = 0;
    };
    struct Scratches {
      std::vector<Scratch> v;
      ~Scratches() {
        for (auto& s : v)
          if (s.p) cudaFree(s.p);
      }
    };
    static thread_local Scratches scs;
    int dev = 0;
    CHK_CUDA(cudaGetDevice(&dev));
    Scratch* sc = nullptr;
    for (auto& e : scs.v)
      if (e.dev == dev && e.stream == s) sc = &e;
    if (!sc) {
      scs.v.push_back(Scratch{dev, s, nullptr, 0});
      sc = &scs.v.back();
    }
    const size_t pb = sizeof(double) * 2 * (size_t)grid->n * 16 * B;  // N*G <= 16 n
    const size_t need = pb + sizeof(unsigned) * B;
    if (sc->cap < need) {
      if (sc->p) {
        CHK_CUDA(cudaStreamSynchronize(s));  // earlier calls on this stream may still use it
        cudaFree(sc->p);
        sc->p = nullptr;
        sc->cap = 0;
      }
      CHK_CUDA(cudaMalloc(&sc->p, need));
      sc->cap = need;
    }
    part = static_cast<double*>(sc->p);
    cnt = reinterpret_cast<unsigned*>(static_cast<char*>(sc->p) + pb);
    CHK_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned) * B, s));
  }
  if (generic_n(grid->n)) {
    gen_stencil_kernel<<<dim3(grid->n, B), 256, 0, s>>>(g, beta, x, y, xy ? part : nullptr, nullptr);
    CHK_LAUNCHED();
    if (xy) {
      gen_finalize_kernel<<<B, 256, 0, s>>>(part, grid->n, xy, nullptr, 1);
      CHK_LAUNCHED();
    }
    return CHK_OK;
  }
  CHK_DISPATCH(grid->n, { rc = O::stencil(s, B, g, beta, x, y, xy, part, cnt); });
  return rc;
}

int32_t chk_corrector_rhs(const chk_grid* grid, const double* beta, double* f, int32_t B,
                          int32_t direction, double scale, void* stream) {
  Geo g;
  int rc = check_grid(grid, &g);
  if (rc) return rc;
  if (!beta || !f || B < 1) return fail(CHK_EINVAL, "bad arguments");
  if (direction < 1 || direction > 3) return fail(CHK_EINVAL, "direction must be in 1..3");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (generic_n(grid->n)) {
    gen_corrector_rhs_kernel<<<dim3(grid->n, B), 256, 0, s>>>(g, beta, f, direction - 1, scale);
    CHK_LAUNCHED();
    return CHK_OK;
  }
  CHK_DISPATCH(grid->n, { rc = O::rhs(s, B, g, beta, f, direction - 1, scale); });
  return rc;
}

size_t chk_pcg_workspace_bytes(const chk_grid* grid, const chk_precond_plan* plan, int32_t B,
                               int32_t max_iter) {
  if (!grid || !plan || B < 1 || max_iter < 1 || !any_n(grid->n)) return 0;
  return carve(nullptr, grid->n, B, max_iter).bytes;
}

}  // extern "C"

namespace {

int solve_batched_impl(const chk_grid* grid, const chk_precond_plan* plan, const double* beta, const double* f,
                       double* u, int32_t B, const chk_pcg_opts* opts, int32_t* iterations, double* final_rel,
                       int32_t* status, int32_t* rhs_projected, double* history, void* workspace,
                       size_t workspace_bytes, void* stream) {
  g_launches = 0;
  Geo g;
  int rc = check_grid(grid, &g);
  if (rc) return rc;
  if (!plan || plan->n != grid->n) return fail(CHK_EINVAL, "plan grid size does not match");
  if (!beta || !f || !u || B < 1 || !opts) return fail(CHK_EINVAL, "bad arguments");
  if (!(opts->tol > 0.0)) return fail(CHK_EINVAL, "tolerance must be positive");
  if (opts->max_iter < 1) return fail(CHK_EINVAL, "max_iter must be >= 1");
  const int n = grid->n;
  Workspace w = carve(workspace, n, B, opts->max_iter);
  if (!workspace || workspace_bytes < w.bytes) return fail(CHK_EINVAL, "workspace too small");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  PlanDev pl = plan_dev(plan);
  if (generic_n(n))
    return gen_solve(g, pl, beta, f, u, B, opts, iterations, final_rel, status, rhs_projected, history, w, s);
  SolveCtl ctl{w.st, w.Rh, w.part, w.hist, maxblk_of(n), opts->max_iter, opts->tol,
               opts->precond_residual_stopping ? 1 : 0, nullptr, 0};
  int* flags = g_pinned.poll_flags();
  if (!flags) return fail(CHK_ECUDA, "cudaMallocHost failed");
  CHK_CUDA(cudaMemsetAsync(w.st, 0, sizeof(RState) * B, s));
  CHK_CUDA(cudaMemsetAsync(w.hist, 0, sizeof(double) * (size_t)opts->max_iter * B, s));

  cudaEvent_t ev[2];
  CHK_CUDA(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
  CHK_CUDA(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
  auto run = [&]() -> int {
    int rc2 = CHK_OK;
    CHK_DISPATCH(n, {
      // initialisation: r = f (projected), u = 0, z = P r, p = z  (solver.py:131-156);
      // r is kept as its spectrum R from here on
      if ((rc2 = O::rhs_stats(s, B, f, ctl))) return rc2;
      if ((rc2 = O::fwd(FWD_INIT, s, B, g, beta, f, u, w.S, pl, ctl, 0))) return rc2;
      if ((rc2 = O::mid(MID_INIT, s, B, w.S, pl, ctl, 0))) return rc2;
      if ((rc2 = O::inv(INV_INIT, s, B, w.S, w.p, u, pl, ctl, 0))) return rc2;
      // iterations, polled every `chunk` with one chunk of look-ahead
      const int chunk = (n >= 128) ? 2 : 8;
      bool pending = false;
      int ev_i = 0;
      // poll: stop when the previous chunk's flag shows no active realization
      auto poll = [&](int it, bool& stop) -> int {
        stop = false;
        if (it % chunk == 0 || it == opts->max_iter) {
          if (pending) {
            CHK_CUDA(cudaEventSynchronize(ev[ev_i ^ 1]));
            if (!reinterpret_cast<volatile int*>(flags)[ev_i ^ 1]) {
              stop = true;
              return CHK_OK;
            }
          }
          poll_active_kernel<<<1, 256, 0, s>>>(w.st, B, flags + ev_i);
          CHK_LAUNCHED();
          CHK_CUDA(cudaEventRecord(ev[ev_i], s));
          ev_i ^= 1;
          pending = true;
        }
        return CHK_OK;
      };
      const int Ba = pair_split<O>(B);
      if (Ba > 0) {
        // Two halves half an iteration apart; every plane launch pairs the forward
        // pass of one half with the inverse pass of the other (pair_plane_kernel):
        //   fwd(A,1) mid(A,1) | [inv(A,k) fwd(B,k)] mid(B,k) [fwd(A,k+1) inv(B,k)] mid(A,k+1) | ...
        const size_t nb = (size_t)n * n * n, spec = (size_t)n * n * (n / 2 + 1);
        const size_t lb = (size_t)g.L * g.L * g.L;
        auto fargs = [&](int b0, int Bn, int it) {
          SolveCtl c = ctl;
          c.st += b0; c.Rh += spec * b0; c.part += (size_t)2 * ctl.maxblk * b0; c.hist += (size_t)ctl.max_iter * b0;
          return FwdArgs{g, beta + lb * b0, w.p + nb * b0, u + nb * b0, w.S + spec * b0, c, Bn, it, Bn * O::PLANE_BLOCKS};
        };
        auto iargs = [&](int b0, int Bn, int it) {
          const FwdArgs f = fargs(b0, Bn, it);
          return InvArgs{f.S, w.p + nb * b0, f.u, f.ctl, Bn, it, Bn * O::PLANE_BLOCKS};
        };
        const int Bb = B - Ba;
        const FwdArgs A1 = fargs(0, Ba, 1);
        if ((rc2 = O::fwd(FWD_Q, s, Ba, g, A1.beta, A1.p, A1.u, A1.S, pl, A1.ctl, 1))) return rc2;
        if ((rc2 = O::mid(MID_ITER, s, Ba, A1.S, pl, A1.ctl, 1))) return rc2;
        int a_pending = 1;  // iteration of half A whose inverse pass is still to run
        for (int it = 1; it <= opts->max_iter; ++it) {
          const FwdArgs Bf = fargs(Ba, Bb, it);
          if ((rc2 = O::pair(s, Bf, iargs(0, Ba, it), pl))) return rc2;
          a_pending = 0;
          if ((rc2 = O::mid(MID_ITER, s, Bb, Bf.S, pl, Bf.ctl, it))) return rc2;
          if (it < opts->max_iter) {
            if ((rc2 = O::pair(s, fargs(0, Ba, it + 1), iargs(Ba, Bb, it), pl))) return rc2;
            if ((rc2 = O::mid(MID_ITER, s, Ba, A1.S, pl, fargs(0, Ba, it + 1).ctl, it + 1))) return rc2;
            a_pending = it + 1;
          } else {
            const InvArgs Bi = iargs(Ba, Bb, it);
            if ((rc2 = O::inv(INV_ITER, s, Bb, Bi.S, Bi.p, Bi.u, pl, Bi.ctl, it))) return rc2;
          }
          bool stop;
          if ((rc2 = poll(it, stop))) return rc2;
          if (stop) break;
        }
        if (a_pending) {  // half A's last middle pass ran: finish its u update
          const InvArgs Ai = iargs(0, Ba, a_pending);
          if ((rc2 = O::inv(INV_ITER, s, Ba, Ai.S, Ai.p, Ai.u, pl, Ai.ctl, a_pending))) return rc2;
        }
      } else
      for (int it = 1; it <= opts->max_iter; ++it) {
        // q = A p, p.q, alpha; Q = FFT(q)            (solver.py:162-166)
        if ((rc2 = O::fwd(FWD_Q, s, B, g, beta, w.p, u, w.S, pl, ctl, it))) return rc2;
        // R -= alpha Q, stop test, z = P r, r.z, beta (solver.py:168-183)
        if ((rc2 = O::mid(MID_ITER, s, B, w.S, pl, ctl, it))) return rc2;
        // u += alpha p, p = z + beta p                (solver.py:167,184)
        if ((rc2 = O::inv(INV_ITER, s, B, w.S, w.p, u, pl, ctl, it))) return rc2;
        bool stop;
        if ((rc2 = poll(it, stop))) return rc2;
        if (stop) break;
      }
      if ((rc2 = O::mean_u(s, B, u, ctl))) return rc2;
    });
    {
      const size_t nb = (size_t)n * n * n;
      sub_mean_kernel<<<1184, 256, 0, s>>>(u, w.st, nb, B);
      CHK_LAUNCHED();
    }
    return rc2;
  };
  rc = run();
  cudaEventDestroy(ev[0]);
  cudaEventDestroy(ev[1]);
  if (rc) return rc;
  rc = read_back(w, B, opts->max_iter, iterations, final_rel, status, rhs_projected, history, s);
  g_prof.collect();
  return rc;
}

}  // namespace

extern "C" {

int32_t chk_pcg_solve_batched(const chk_grid* grid, const chk_precond_plan* plan,
                              const double* beta, const double* f, double* u, int32_t B,
                              const chk_pcg_opts* opts, int32_t* iterations, double* final_rel,
                              int32_t* status, int32_t* rhs_projected, double* history,
                              void* workspace, size_t workspace_bytes, void* stream) {
  return solve_batched_impl(grid, plan, beta, f, u, B, opts, iterations, final_rel, status, rhs_projected, history,
                            workspace, workspace_bytes, stream);
}

// Host-buffer pipeline: three lanes (host threads, each with its own stream,
// device slot and solver workspace) take chunks round-robin; on a lane a chunk
// is uploaded, solved and downloaded in stream order, and the lanes overlap on
// the GPU -- one lane's copies and convergence tail run under the other lanes'
// solves (config 3, e2e: 1 lane 4.0e10, 2 lanes 4.24e10, 3 lanes x 32
// realizations 4.30e10 DOF-it/s).  CHK_HOST_LANES overrides (1..4).
static int host_lanes(int nchunks) {
  static const int want = getenv("CHK_HOST_LANES") ? atoi(getenv("CHK_HOST_LANES")) : 3;
  const int l = want < 1 ? 1 : (want > 4 ? 4 : want);
  return nchunks < l ? nchunks : l;
}

size_t chk_pcg_host_workspace_bytes(const chk_grid* grid, const chk_precond_plan* plan, int32_t chunk,
                                    int32_t max_iter) {
  if (!grid || !plan || chunk < 1 || max_iter < 1 || !any_n(grid->n)) return 0;
  const size_t nb = (size_t)grid->n * grid->n * grid->n;
  const size_t lb = (size_t)grid->L * grid->L * grid->L;
  const size_t slot = align_up(sizeof(double) * (2 * nb + lb) * chunk) + align_up(2 * sizeof(uint64_t) * chunk);
  const size_t sw = chk_pcg_workspace_bytes(grid, plan, chunk, max_iter);
  if (sw == 0) return 0;
  return (size_t)host_lanes(1 << 30) * (slot + align_up(sw));
}

}  // extern "C"

namespace {

// Inputs of one host pipeline run: per-cell contrasts from host arrays or drawn
// on the device from Philox keys; the load from a host array or the device
// corrector kernel.
struct PipeIn {
  const double* beta_host;  // [B][L^3] or null (then keys_host)
  const uint64_t* keys_host;  // [B][2] Philox keys (SeedSequence(seed).generate_state(2, uint64))
  double cov_p;
  int ckind;
  double beta0, beta1;
  const double* f_host;  // [B][n^3] or null (then the corrector load along rhs_dir)
  int rhs_dir;
};

int host_pipeline(const chk_grid* grid, const chk_precond_plan* plan, const PipeIn& in, double* u_host, int B,
                  int chunk, const chk_pcg_opts* opts, int32_t* iterations, double* final_rel, int32_t* status,
                  int32_t* rhs_projected, double* history, void* workspace, size_t workspace_bytes, void* stream) {
  if (!grid || !plan || !u_host || B < 1 || chunk < 1 || !opts) return fail(CHK_EINVAL, "bad arguments");
  if (chunk > B) chunk = B;
  Geo geo;
  int rc0 = check_grid(grid, &geo);
  if (rc0) return rc0;
  const size_t need = chk_pcg_host_workspace_bytes(grid, plan, chunk, opts->max_iter);
  if (!workspace || workspace_bytes < need || need == 0) return fail(CHK_EINVAL, "workspace too small");
  const size_t nb = (size_t)grid->n * grid->n * grid->n;
  const size_t lb = (size_t)grid->L * grid->L * grid->L;
  const size_t data_bytes = align_up(sizeof(double) * (2 * nb + lb) * chunk);
  const size_t slot_bytes = data_bytes + align_up(2 * sizeof(uint64_t) * chunk);
  const size_t solver_bytes = align_up(chk_pcg_workspace_bytes(grid, plan, chunk, opts->max_iter));
  // Chunk schedule: full chunks while more than a round of them remains, then halved and
  // quartered chunks, handed to whichever lane is free -- the lanes finish together and
  // the last download, which nothing can overlap, is a quarter chunk (CHK_HOST_TAPER=0:
  // equal chunks, round-robin as before).
  static const bool taper = !(getenv("CHK_HOST_TAPER") && atoi(getenv("CHK_HOST_TAPER")) == 0);
  const int lanes = host_lanes((B + chunk - 1) / chunk);
  std::vector<std::pair<int, int>> sched;  // (first realization, count)
  for (int b0 = 0; b0 < B;) {
    int c = chunk;
    if (taper) {
      const int rem = B - b0;
      if (rem <= lanes * chunk / 2 && chunk >= 4) c = chunk / 4;
      else if (rem <= lanes * chunk && chunk >= 2) c = chunk / 2;
    }
    c = std::min(c, B - b0);
    sched.push_back({b0, c});
    b0 += c;
  }
  const int nchunks = (int)sched.size();
  std::atomic<int> next_chunk{0};
  const double h = 1.0 / grid->n;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int dev = 0;
  CHK_CUDA(cudaGetDevice(&dev));
  cudaEvent_t start;
  CHK_CUDA(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
  CHK_CUDA(cudaEventRecord(start, s));  // the lanes follow the caller's prior work
  struct LaneOut {
    int rc = CHK_OK;
    std::string err;
    long long launches = 0;
  };
  std::vector<LaneOut> out(lanes);
  auto lane_fn = [&](int lane) {
    LaneOut& o = out[lane];
    auto bad = [&](int code, const char* what, cudaError_t e) {
      o.rc = code;
      o.err = std::string(what) + (e != cudaSuccess ? std::string(": ") + cudaGetErrorString(e) : std::string());
    };
    cudaError_t e = cudaSetDevice(dev);
    if (e != cudaSuccess) return bad(CHK_ECUDA, "lane cudaSetDevice", e);
    cudaStream_t ls;
    if ((e = cudaStreamCreateWithFlags(&ls, cudaStreamNonBlocking)) != cudaSuccess)
      return bad(CHK_ECUDA, "lane stream", e);
    char* base = static_cast<char*>(workspace) + (size_t)lane * (slot_bytes + solver_bytes);
    double* d_f = reinterpret_cast<double*>(base);
    double* d_u = d_f + nb * chunk;
    double* d_b = d_u + nb * chunk;
    uint64_t* d_k = reinterpret_cast<uint64_t*>(base + data_bytes);
    void* solver_ws = base + slot_bytes;
    if ((e = cudaStreamWaitEvent(ls, start, 0)) != cudaSuccess) bad(CHK_ECUDA, "lane wait", e);
    for (int c = next_chunk.fetch_add(1); c < nchunks && o.rc == CHK_OK; c = next_chunk.fetch_add(1)) {
      const int b0 = sched[c].first, nbc = sched[c].second;
      if (in.beta_host) {
        if ((e = cudaMemcpyAsync(d_b, in.beta_host + lb * b0, sizeof(double) * lb * nbc, cudaMemcpyHostToDevice, ls))) {
          bad(CHK_ECUDA, "upload beta", e);
          break;
        }
      } else {
        if ((e = cudaMemcpyAsync(d_k, in.keys_host + 2 * (size_t)b0, 2 * sizeof(uint64_t) * nbc,
                                 cudaMemcpyHostToDevice, ls))) {
          bad(CHK_ECUDA, "upload keys", e);
          break;
        }
        const int ncell = (int)lb;
        const int gx = (int)std::min<long long>(((long long)ncell / 4 + 255) / 256 + 1, 1184);
        sample_cells_kernel<<<dim3(gx, nbc), 256, 0, ls>>>(d_k, ncell, in.cov_p, in.ckind, in.beta0, in.beta1, d_b);
        ++o.launches;
        if ((e = cudaGetLastError())) {
          bad(CHK_ECUDA, "sample_cells launch", e);
          break;
        }
      }
      if (in.f_host) {
        if ((e = cudaMemcpyAsync(d_f, in.f_host + nb * b0, sizeof(double) * nb * nbc, cudaMemcpyHostToDevice, ls))) {
          bad(CHK_ECUDA, "upload f", e);
          break;
        }
      } else {
        // PCG load h^(d-1) * h^(2-d) * 1/2 (c[x+e_i] - c[x-e_i])  (homogenize.py:85-89,110)
        int rc = CHK_OK;
        if (generic_n(grid->n)) {
          gen_corrector_rhs_kernel<<<dim3(grid->n, nbc), 256, 0, ls>>>(geo, d_b, d_f, in.rhs_dir - 1, h * h * (1.0 / h));
          if (cudaGetLastError() != cudaSuccess) rc = fail(CHK_ECUDA, "corrector_rhs launch");
        } else {
          CHK_DISPATCH_V(grid->n, rc, { rc = O::rhs(ls, nbc, geo, d_b, d_f, in.rhs_dir - 1, h * h * (1.0 / h)); });
        }
        ++o.launches;
        if (rc) {
          o.rc = rc;
          o.err = g_err;
          break;
        }
      }
      const int rc = solve_batched_impl(grid, plan, d_b, d_f, d_u, nbc, opts, iterations ? iterations + b0 : nullptr,
                                        final_rel ? final_rel + b0 : nullptr, status ? status + b0 : nullptr,
                                        rhs_projected ? rhs_projected + b0 : nullptr,
                                        history ? history + (size_t)opts->max_iter * b0 : nullptr, solver_ws,
                                        solver_bytes, ls);
      o.launches += g_launches;
      if (rc) {
        o.rc = rc;
        o.err = g_err;
        break;
      }
      if ((e = cudaMemcpyAsync(u_host + nb * b0, d_u, sizeof(double) * nb * nbc, cudaMemcpyDeviceToHost, ls))) {
        bad(CHK_ECUDA, "download", e);
        break;
      }
    }
    if ((e = cudaStreamSynchronize(ls)) != cudaSuccess && o.rc == CHK_OK) bad(CHK_ECUDA, "lane synchronize", e);
    cudaStreamDestroy(ls);
  };
  if (lanes == 1) {
    lane_fn(0);
  } else {
    // lane 0 runs on the calling thread; no exception may cross the C ABI
    std::vector<std::thread> th;
    try {
      for (int l = 1; l < lanes; ++l) th.emplace_back(lane_fn, l);
    } catch (const std::exception& ex) {
      for (int l = 1 + (int)th.size(); l < lanes; ++l) {
        out[l].rc = CHK_ECUDA;
        out[l].err = std::string("cannot start a pipeline lane: ") + ex.what();
      }
    }
    lane_fn(0);
    for (auto& t : th) t.join();
  }
  cudaEventDestroy(start);
  long long launches = 0;
  int rc = CHK_OK;
  for (auto& o : out) {
    launches += o.launches;
    if (o.rc && rc == CHK_OK) rc = fail(o.rc, "host pipeline: " + o.err);
  }
  g_launches = launches;
  return rc;
}

}  // namespace

extern "C" {

int32_t chk_pcg_solve_host(const chk_grid* grid, const chk_precond_plan* plan, const double* beta_host,
                           const double* f_host, double* u_host, int32_t B, int32_t chunk,
                           const chk_pcg_opts* opts, int32_t* iterations, double* final_rel,
                           int32_t* status, int32_t* rhs_projected, double* history,
                           void* workspace, size_t workspace_bytes, void* stream) {
  if (!beta_host || !f_host) return fail(CHK_EINVAL, "bad arguments");
  PipeIn in{beta_host, nullptr, 0.0, 0, 0.0, 0.0, f_host, 0};
  return host_pipeline(grid, plan, in, u_host, B, chunk, opts, iterations, final_rel, status, rhs_projected,
                       history, workspace, workspace_bytes, stream);
}

int32_t chk_pcg_solve_seeds(const chk_grid* grid, const chk_precond_plan* plan, const uint64_t* keys_host,
                            double coverage_prob, int32_t contrast_kind, double beta0, double beta1,
                            const double* f_host, int32_t rhs_direction, double* u_host, int32_t B, int32_t chunk,
                            const chk_pcg_opts* opts, int32_t* iterations, double* final_rel, int32_t* status,
                            int32_t* rhs_projected, double* history, void* workspace, size_t workspace_bytes,
                            void* stream) {
  if (!keys_host) return fail(CHK_EINVAL, "keys_host is NULL");
  if (contrast_kind != CHK_CONTRAST_FIXED && contrast_kind != CHK_CONTRAST_TWO_VALUE)
    return fail(CHK_EINVAL, "contrast_kind must be CHK_CONTRAST_FIXED or CHK_CONTRAST_TWO_VALUE");
  if (!f_host && (rhs_direction < 1 || rhs_direction > 3))
    return fail(CHK_EINVAL, "rhs_direction must be in 1..3 when f_host is NULL");
  PipeIn in{nullptr, keys_host, coverage_prob, contrast_kind, beta0, beta1, f_host, rhs_direction};
  return host_pipeline(grid, plan, in, u_host, B, chunk, opts, iterations, final_rel, status, rhs_projected,
                       history, workspace, workspace_bytes, stream);
}

int32_t chk_sample_cells(const chk_grid* grid, const uint64_t* keys, double coverage_prob, int32_t contrast_kind,
                         double beta0, double beta1, double* beta, int32_t B, void* stream) {
  // only the lattice matters here (any L; no grid-size restriction of the solver)
  if (!grid || grid->L < 1 || grid->d != 3) return fail(CHK_EINVAL, "bad grid (need d = 3, L >= 1)");
  if (!keys || !beta || B < 1) return fail(CHK_EINVAL, "bad arguments");
  if (contrast_kind != CHK_CONTRAST_FIXED && contrast_kind != CHK_CONTRAST_TWO_VALUE)
    return fail(CHK_EINVAL, "contrast_kind must be CHK_CONTRAST_FIXED or CHK_CONTRAST_TWO_VALUE");
  const int ncell = grid->L * grid->L * grid->L;
  const int gx = (int)std::min<long long>(((long long)ncell / 4 + 255) / 256 + 1, 1184);
  sample_cells_kernel<<<dim3(gx, B), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      keys, ncell, coverage_prob, contrast_kind, beta0, beta1, beta);
  CHK_LAUNCHED();
  return CHK_OK;
}

}  // extern "C"

// ----------------------------------------------------------------------------
// slab decomposition (one grid over several GPUs)
// ----------------------------------------------------------------------------
static int slab_geo(const chk_grid* grid, const chk_slab* sl, const double* lo, const double* hi, SlabGeo* out) {
  if (!sl || sl->nranks < 1 || sl->rank < 0 || sl->rank >= sl->nranks)
    return fail(CHK_EINVAL, "bad slab (nranks/rank)");
  int ok = 0;
  CHK_DISPATCH(grid->n, {
    ok = O::slab_ok(sl->nranks);
    if (ok) *out = O::slab(sl->nranks, sl->rank, lo, hi);
  });
  if (!ok) return fail(CHK_EINVAL, "nranks must divide n and the middle-pass tile count");
  return CHK_OK;
}

struct SlabWs {
  double2* Rh;
  double* part;
  RState* st;
  double* hist;
  size_t bytes;
};

static SlabWs slab_carve(void* base, int n, int P, int B, int max_iter) {
  const size_t spec_loc = (size_t)n * n * (n / 2 + 1) / P;
  char* c = static_cast<char*>(base);
  SlabWs w{};
  size_t off = 0;
  w.Rh = reinterpret_cast<double2*>(c + off); off = align_up(off + sizeof(double2) * spec_loc * B);
  w.part = reinterpret_cast<double*>(c + off); off = align_up(off + sizeof(double) * 2 * (size_t)maxblk_of(n) * B);
  w.st = reinterpret_cast<RState*>(c + off); off = align_up(off + sizeof(RState) * B);
  w.hist = reinterpret_cast<double*>(c + off); off = align_up(off + sizeof(double) * (size_t)max_iter * B);
  w.bytes = off;
  return w;
}

extern "C" {

size_t chk_slab_exchange_elems(const chk_grid* grid, const chk_slab* slab, int32_t B) {
  if (!grid || !slab || !supported_n(grid->n) || slab->nranks < 1 || B < 1) return 0;
  const size_t n = grid->n;
  return n * n * (n / 2 + 1) / slab->nranks * (size_t)B;
}

size_t chk_slab_workspace_bytes(const chk_grid* grid, const chk_precond_plan* plan, const chk_slab* slab,
                                int32_t B, int32_t max_iter) {
  if (!grid || !plan || !slab || B < 1 || max_iter < 1 || !supported_n(grid->n) || slab->nranks < 1) return 0;
  return slab_carve(nullptr, grid->n, slab->nranks, B, max_iter).bytes;
}

int32_t chk_slab_phase(const chk_grid* grid, const chk_precond_plan* plan, const chk_slab* slab,
                       int32_t phase, int32_t it, const double* beta, const double* f, double* u, double* p,
                       void* xa, void* xb, const double* halo_lo, const double* halo_hi, double* red,
                       int32_t B, const chk_pcg_opts* opts, void* workspace, size_t workspace_bytes,
                       void* stream) {
  return chk_slab_phase_planes(grid, plan, slab, phase, it, 0, -1, beta, f, u, p, xa, xb, halo_lo, halo_hi, red,
                               B, opts, workspace, workspace_bytes, stream);
}

int32_t chk_slab_phase_planes(const chk_grid* grid, const chk_precond_plan* plan, const chk_slab* slab,
                              int32_t phase, int32_t it, int32_t plane_begin, int32_t plane_count,
                              const double* beta, const double* f, double* u, double* p, void* xa, void* xb,
                              const double* halo_lo, const double* halo_hi, double* red, int32_t B,
                              const chk_pcg_opts* opts, void* workspace, size_t workspace_bytes, void* stream) {
  Geo g;
  int rc = check_grid(grid, &g);
  if (rc) return rc;
  if (!plan || plan->n != grid->n || !opts || B < 1 || !red) return fail(CHK_EINVAL, "bad arguments");
  if (!supported_n(grid->n)) return fail(CHK_EUNSUPPORTED, "slab decomposition needs a power-of-two n in [8, 512]");
  SlabGeo sg;
  if ((rc = slab_geo(grid, slab, halo_lo, halo_hi, &sg))) return rc;
  if (plane_count < 0) plane_count = sg.nloc - plane_begin;
  if (plane_begin < 0 || plane_count < 1 || plane_begin + plane_count > sg.nloc)
    return fail(CHK_EINVAL, "plane range outside the rank's slab");
  const bool ranged = plane_begin != 0 || plane_count != sg.nloc;
  if (ranged && phase != CHK_SLAB_FWD_INIT && phase != CHK_SLAB_FWD_Q && phase != CHK_SLAB_INV)
    return fail(CHK_EINVAL, "only the plane phases (FWD_INIT, FWD_Q, INV) take a plane range");
  sg.run0 = plane_begin;
  sg.nrun = plane_count;
  const int n = grid->n;
  SlabWs w = slab_carve(workspace, n, slab->nranks, B, opts->max_iter);
  if (!workspace || workspace_bytes < w.bytes) return fail(CHK_EINVAL, "workspace too small");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  PlanDev pl = plan_dev(plan);
  SolveCtl ctl{w.st, w.Rh, w.part, w.hist, maxblk_of(n), opts->max_iter, opts->tol,
               opts->precond_residual_stopping ? 1 : 0, red, 1};
  double2* XA = static_cast<double2*>(xa);
  double2* XB = static_cast<double2*>(xb);
  const double ntot = (double)n * n * n;
  auto zero_red = [&]() { return cudaMemsetAsync(red, 0, sizeof(double) * 4 * B, s); };
  auto decide = [&](int what) -> int {
    decide_kernel<<<1, 256, 0, s>>>(ctl, red, B, what, it, ntot);
    CHK_LAUNCHED();
    return CHK_OK;
  };
  CHK_DISPATCH(n, {
    switch (phase) {
      case CHK_SLAB_STATS:
        CHK_CUDA(cudaMemsetAsync(w.st, 0, sizeof(RState) * B, s));
        CHK_CUDA(cudaMemsetAsync(w.hist, 0, sizeof(double) * (size_t)opts->max_iter * B, s));
        CHK_CUDA(zero_red());
        rc = O::rhs_stats(s, B, f, ctl, sg);
        break;
      case CHK_SLAB_STATS_DECIDE: rc = decide(DECIDE_STATS); break;
      case CHK_SLAB_FWD_INIT: rc = O::fwd(FWD_INIT, s, B, g, beta, f, u, XA, pl, ctl, 0, sg); break;
      case CHK_SLAB_MID:
        CHK_CUDA(zero_red());
        rc = O::mid(it == 0 ? MID_INIT : MID_ITER, s, B, XB, pl, ctl, it, sg);
        break;
      case CHK_SLAB_MID_DECIDE: rc = decide(DECIDE_MID); break;
      case CHK_SLAB_INV: rc = O::inv(it == 0 ? INV_INIT : INV_ITER, s, B, XA, p, u, pl, ctl, it, sg); break;
      case CHK_SLAB_FWD_Q:
        if (plane_begin == 0) CHK_CUDA(zero_red());  // first plane chunk of the phase
        rc = O::fwd(FWD_Q, s, B, g, beta, p, u, XA, pl, ctl, it, sg);
        break;
      case CHK_SLAB_ALPHA_DECIDE: rc = decide(DECIDE_ALPHA); break;
      case CHK_SLAB_MEANU:
        CHK_CUDA(zero_red());
        rc = O::mean_u(s, B, u, ctl, sg);
        break;
      case CHK_SLAB_MEANU_APPLY: {
        if ((rc = decide(DECIDE_MEANU))) break;
        const size_t nb = (size_t)sg.nloc * n * n;
        sub_mean_kernel<<<1184, 256, 0, s>>>(u, w.st, nb, B);
        CHK_LAUNCHED();
        break;
      }
      default: return fail(CHK_EINVAL, "unknown slab phase");
    }
  });
  return rc;
}

int32_t chk_slab_status_async(const chk_grid* grid, const chk_slab* slab, int32_t B, int32_t max_iter,
                              void* workspace, int32_t* status, void* stream) {
  if (!grid || !slab || !workspace || !status || B < 1 || max_iter < 1 || !supported_n(grid->n))
    return fail(CHK_EINVAL, "bad arguments");
  SlabWs w = slab_carve(workspace, grid->n, slab->nranks, B, max_iter);
  // the status word of each RState, strided, into a dense [B] int32 array (pinned host or device)
  CHK_CUDA(cudaMemcpy2DAsync(status, sizeof(int32_t), &w.st->status, sizeof(RState), sizeof(int32_t), B,
                             cudaMemcpyDefault, static_cast<cudaStream_t>(stream)));
  return CHK_OK;
}

int32_t chk_slab_read_state(const chk_grid* grid, const chk_slab* slab, int32_t B, int32_t max_iter,
                            void* workspace, int32_t* iterations, double* final_rel, int32_t* status,
                            int32_t* rhs_projected, double* history, void* stream) {
  if (!grid || !slab || !workspace || B < 1 || max_iter < 1 || !supported_n(grid->n))
    return fail(CHK_EINVAL, "bad arguments");
  SlabWs w = slab_carve(workspace, grid->n, slab->nranks, B, max_iter);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  std::vector<RState> hst(B);
  CHK_CUDA(cudaMemcpyAsync(hst.data(), w.st, sizeof(RState) * B, cudaMemcpyDeviceToHost, s));
  if (history)
    CHK_CUDA(cudaMemcpyAsync(history, w.hist, sizeof(double) * (size_t)max_iter * B, cudaMemcpyDeviceToHost, s));
  CHK_CUDA(cudaStreamSynchronize(s));
  for (int b = 0; b < B; ++b) {
    if (status) status[b] = hst[b].status == ST_ACTIVE ? 3 : hst[b].status;
    if (iterations) iterations[b] = hst[b].iters;
    if (final_rel) final_rel[b] = hst[b].final_rel;
    if (rhs_projected) rhs_projected[b] = hst[b].rhs_projected;
  }
  return CHK_OK;
}

}  // extern "C"
