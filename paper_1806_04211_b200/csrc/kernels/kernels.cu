// kernels.cu -- SIMT kernels of the GF(p) path for sm_100a:
//   K1 (small-K SIMT contraction, the K<=~32 class of UpdateRow / ClearDown),
//   K3/K4 (row/column gather, riffle, zero-riffle, identity planting),
//   K2 base case (single-CTA Gauss-Jordan ECH in shared memory),
//   K6 (counter-form SplitMix64 generator).
// The tensor-core contraction lives in gf_mad_tc.cu.
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <atomic>
#include <mutex>
#include <vector>

#include "../common.hpp"
#include "kernels.hpp"

namespace gfq::dev {

bool pdl_enabled() {
  static const bool on = std::getenv("GFQ_NO_PDL") == nullptr;
  return on;
}

// ------------------------------------------------------------------ helpers
// x mod p for any 32-bit x: q_est = floor(x * ceil(2^32/p) / 2^32) is q or q+1.
__device__ __forceinline__ std::uint32_t modp(std::uint32_t x, std::uint32_t p,
                                              std::uint32_t magic) {
  const std::uint32_t q = __umulhi(x, magic);
  const std::int32_t r = static_cast<std::int32_t>(x - q * p);
  return static_cast<std::uint32_t>(r < 0 ? r + static_cast<std::int32_t>(p) : r);
}

static inline std::uint32_t magic_of(std::uint32_t p) {
  return static_cast<std::uint32_t>((0x100000000ULL / p) + 1);
}

// Largest K chunk for which sum_{t<k} (p-1)^2 + (p-1) stays below 2^31.
static inline std::int64_t k_chunk_limit(std::uint32_t p) {
  const std::uint64_t sq = std::uint64_t(p - 1) * (p - 1);
  if (sq == 0) return std::int64_t(1) << 40;
  const std::uint64_t lim = (0x7FFFFFFFULL - p) / sq;
  return static_cast<std::int64_t>(lim / 128 * 128 > 0 ? lim / 128 * 128 : lim);
}

// ------------------------------------------------------------------ K1 SIMT
namespace {
constexpr int kTm = 64, kTn = 64, kTk = 32;

__global__ void __launch_bounds__(256)
mad_simt_kernel(std::uint32_t p, std::uint32_t magic, int m, int n, int k,
                const std::uint8_t* __restrict__ A, std::int64_t lda,
                const std::uint8_t* __restrict__ B, std::int64_t ldb,
                const std::uint8_t* Cin, std::int64_t ldc, std::uint8_t* D,
                std::int64_t ldd) {
  pdl_wait_and_release();
  __shared__ std::uint8_t As[kTm][kTk + 4];
  __shared__ std::uint8_t Bs[kTk][kTn + 4];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int m0 = blockIdx.y * kTm, n0 = blockIdx.x * kTn;
  std::uint32_t acc[4][4] = {};
  for (int k0 = 0; k0 < k; k0 += kTk) {
    // 64x32 A tile and 32x64 B tile, 8 bytes per thread each.
    for (int e = threadIdx.x; e < kTm * kTk; e += 256) {
      const int r = e / kTk, c = e % kTk;
      const int gr = m0 + r, gc = k0 + c;
      As[r][c] = (gr < m && gc < k) ? A[std::int64_t(gr) * lda + gc] : 0;
    }
    for (int e = threadIdx.x; e < kTk * kTn; e += 256) {
      const int r = e / kTn, c = e % kTn;
      const int gr = k0 + r, gc = n0 + c;
      Bs[r][c] = (gr < k && gc < n) ? B[std::int64_t(gr) * ldb + gc] : 0;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < kTk; ++kk) {
      std::uint32_t a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[ty + 16 * i][kk];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] += a[i] * b[j];
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gr = m0 + ty + 16 * i;
    if (gr >= m) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gc = n0 + tx + 16 * j;
      if (gc >= n) continue;
      std::uint32_t v = acc[i][j];
      if (Cin) v += Cin[std::int64_t(gr) * ldc + gc];
      D[std::int64_t(gr) * ldd + gc] = static_cast<std::uint8_t>(modp(v, p, magic));
    }
  }
}

// Small-K contraction (K <= 32): the rank-r' updates of UpdateRow /
// ClearDown when a block row contributes few new pivots (the
// K in 1..7 class).  HBM-bound: each thread owns 16 consecutive outputs of
// one row (one uint4 of D and of Cin), the K coefficients of its A row and
// the K x 16-byte slab of B (both L1/L2 resident across threads).
constexpr int kSmallK = 32;
// MAPS: the row maps of the fused gather / riffle forms (mad_smallk_maps):
// B row t = Bsrc[brm[t]], the addend of output row i = Cin[crm[i]] (-1:
// none), output row i lands at D[drm[i]].
struct SmallkMaps {
  const std::int32_t* brm;
  const std::int32_t* crm;
  const std::int32_t* drm;
};
template <bool MAPS>
__global__ void __launch_bounds__(256)
mad_smallk_kernel(std::uint32_t p, std::uint32_t magic, int m, int n, int k,
                  const std::uint8_t* __restrict__ A, std::int64_t lda,
                  const std::uint8_t* __restrict__ B, std::int64_t ldb,
                  const std::uint8_t* Cin, std::int64_t ldc, std::uint8_t* D, std::int64_t ldd,
                  SmallkMaps mp) {
  pdl_wait_and_release();
  const int nvec = (n + 15) >> 4;
  const std::int64_t tid = std::int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const std::int64_t total = std::int64_t(m) * nvec;
  for (std::int64_t e = tid; e < total; e += std::int64_t(gridDim.x) * blockDim.x) {
    const int i = int(e / nvec), v = int(e % nvec);
    const int j0 = v << 4;
    const bool full = j0 + 16 <= n;
    const std::uint8_t* arow = A + std::int64_t(i) * lda;
    std::uint32_t acc[16];
    if (p == 2) {
      uint4 x = make_uint4(0, 0, 0, 0);
      for (int t = 0; t < k; ++t) {
        if (!arow[t]) continue;
        const std::uint8_t* brow = B + std::int64_t(MAPS && mp.brm ? mp.brm[t] : t) * ldb + j0;
        uint4 b;
        if (full) {
          b = *reinterpret_cast<const uint4*>(brow);
        } else {
          std::uint32_t w[4] = {0, 0, 0, 0};
          for (int c = 0; c < n - j0; ++c) w[c >> 2] |= std::uint32_t(brow[c]) << (8 * (c & 3));
          b = make_uint4(w[0], w[1], w[2], w[3]);
        }
        x.x ^= b.x;
        x.y ^= b.y;
        x.z ^= b.z;
        x.w ^= b.w;
      }
      const std::uint32_t xw[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
      for (int c = 0; c < 16; ++c) acc[c] = (xw[c >> 2] >> (8 * (c & 3))) & 1;
    } else {
#pragma unroll
      for (int c = 0; c < 16; ++c) acc[c] = 0;
      for (int t = 0; t < k; ++t) {
        const std::uint32_t a = arow[t];
        if (!a) continue;
        const std::uint8_t* brow = B + std::int64_t(MAPS && mp.brm ? mp.brm[t] : t) * ldb + j0;
        if (full) {
          const uint4 b = *reinterpret_cast<const uint4*>(brow);
          const std::uint32_t bw[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
          for (int c = 0; c < 16; ++c) acc[c] += a * ((bw[c >> 2] >> (8 * (c & 3))) & 0xFF);
        } else {
          for (int c = 0; c < n - j0; ++c) acc[c] += a * brow[c];
        }
      }
    }
    const std::int64_t ci = MAPS && mp.crm ? std::int64_t(mp.crm[i]) : std::int64_t(i);
    const std::int64_t di = MAPS && mp.drm ? std::int64_t(mp.drm[i]) : std::int64_t(i);
    const std::uint8_t* crow = (Cin && ci >= 0) ? Cin + ci * ldc + j0 : nullptr;
    std::uint8_t* drow = D + di * ldd + j0;
    if (full) {
      std::uint32_t cw[4] = {0, 0, 0, 0};
      if (crow) {
        const uint4 cv = *reinterpret_cast<const uint4*>(crow);
        cw[0] = cv.x;
        cw[1] = cv.y;
        cw[2] = cv.z;
        cw[3] = cv.w;
      }
      std::uint32_t ow[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        std::uint32_t word = 0;
#pragma unroll
        for (int by = 0; by < 4; ++by) {
          const std::uint32_t x = acc[4 * q + by] + ((cw[q] >> (8 * by)) & 0xFF);
          word |= (p == 2 ? (x & 1) : modp(x, p, magic)) << (8 * by);
        }
        ow[q] = word;
      }
      *reinterpret_cast<uint4*>(drow) = make_uint4(ow[0], ow[1], ow[2], ow[3]);
    } else {
      for (int c = 0; c < n - j0; ++c) {
        const std::uint32_t x = acc[c] + (crow ? crow[c] : 0);
        drow[c] = std::uint8_t(modp(x, p, magic));
      }
    }
  }
}

// D = Cin (or 0) for the k == 0 contraction.
}  // namespace

void mad_simt(std::uint32_t p, std::int64_t m, std::int64_t n, std::int64_t k,
              const std::uint8_t* A, std::int64_t lda, const std::uint8_t* B,
              std::int64_t ldb, const std::uint8_t* Cin, std::int64_t ldc,
              std::uint8_t* D, std::int64_t ldd, cudaStream_t s) {
  if (m == 0 || n == 0) return;
  if (k == 0) {
    // D = Cin or 0: a strided copy / fill, as kernels (a copy-engine
    // transfer would queue behind a bulk host copy on the same engine)
    if (Cin == D && ldc == ldd) return;
    if (Cin)
      select2d(D, ldd, m, n, Cin, ldc, nullptr, 0, nullptr, nullptr, s);
    else
      fill2d(D, ldd, m, n, 0, s);
    return;
  }
  const std::int64_t kc = k_chunk_limit(p);
  const std::uint32_t mg = magic_of(p);
  for (std::int64_t k0 = 0; k0 < k; k0 += kc) {
    const std::int64_t kk = (k - k0) < kc ? (k - k0) : kc;
    const std::uint8_t* cin = k0 == 0 ? Cin : D;
    const std::int64_t ldcin = k0 == 0 ? ldc : ldd;
    for (std::int64_t m0 = 0; m0 < m; m0 += std::int64_t(65535) * kTm) {
      const std::int64_t mm = (m - m0) < std::int64_t(65535) * kTm ? (m - m0) : std::int64_t(65535) * kTm;
      dim3 grid(unsigned((n + kTn - 1) / kTn), unsigned((mm + kTm - 1) / kTm));
      GFQ_CUDA(launch_pdl(mad_simt_kernel, dim3(grid), dim3(256), 0, s, 
          p, mg, int(mm), int(n), int(kk), A + m0 * lda + k0, lda, B + k0 * ldb, ldb,
          cin ? cin + m0 * ldcin : nullptr, ldcin, D + m0 * ldd, ldd));
      GFQ_CUDA(cudaGetLastError());
    count_launch();
    }
  }
}

namespace {
std::atomic<int> g_policy{0};
std::atomic<std::int64_t> g_simt{0}, g_tc{0};
std::atomic<std::int64_t> g_launches{0};
std::atomic<bool> g_profile{false};
struct ProfRec {
  cudaEvent_t e0, e1;
  double ops;
  int path;
  const char* task = nullptr;  // issuing task (developer dump)
};
std::mutex g_prof_mtx;
std::vector<ProfRec> g_prof;
}  // namespace

void count_launch(std::int64_t n) { g_launches += n; }
std::int64_t launch_count(bool reset) {
  return reset ? g_launches.exchange(0) : g_launches.load();
}
void set_profile(bool on) { g_profile = on; }
bool profile_on() { return g_profile; }

ProfScope::ProfScope(int kind, double work, cudaStream_t s) : work_(work), kind_(kind), s_(s) {
  if (!g_profile) return;
  GFQ_CUDA(cudaEventCreate(&e0_));
  GFQ_CUDA(cudaEventCreate(&e1_));
  GFQ_CUDA(cudaEventRecord(e0_, s_));
}
ProfScope::~ProfScope() {
  if (!e0_) return;
  cudaEventRecord(e1_, s_);
  std::lock_guard<std::mutex> lk(g_prof_mtx);
  g_prof.push_back(ProfRec{e0_, e1_, work_, kind_, hprof::t_task_name});
}

void profile_take_kinds(int n, std::int64_t* launches, double* work, double* ms, double* union_ms) {
  std::vector<ProfRec> recs;
  {
    std::lock_guard<std::mutex> lk(g_prof_mtx);
    recs.swap(g_prof);
  }
  for (int q = 0; q < n; ++q) {
    launches[q] = 0;
    work[q] = 0;
    ms[q] = 0;
    if (union_ms) union_ms[q] = 0;
  }
  // per family: the launches' [start, end) on a common device clock (the
  // first record's start), merged -- the time the family was running at
  // all, so concurrent launches on several streams are not double counted
  std::vector<std::vector<std::pair<double, double>>> iv(std::size_t(n > 0 ? n : 0));
  for (auto& r : recs) {
    float t = 0, t0 = 0;
    GFQ_CUDA(cudaEventSynchronize(r.e1));
    GFQ_CUDA(cudaEventElapsedTime(&t, r.e0, r.e1));
    if (r.path < n) {
      launches[r.path] += 1;
      work[r.path] += r.ops;
      ms[r.path] += t;
      if (union_ms && cudaEventElapsedTime(&t0, recs.front().e0, r.e0) == cudaSuccess)
        iv[std::size_t(r.path)].emplace_back(double(t0), double(t0) + double(t));
    }
  }
  // developer dump of every launch window (GFQ_PROF_DUMP=path): family,
  // start ms, end ms on the common clock
  if (const char* path = std::getenv("GFQ_PROF_DUMP")) {
    if (FILE* fh = std::fopen(path, "a")) {
      for (int q = 0; q < n; ++q)
        for (const auto& [a, b] : iv[std::size_t(q)]) std::fprintf(fh, "%d %.4f %.4f\n", q, a, b);
      // (GFQ_PROF_DUMP_TASKS: one line per launch with its issuing task)
      if (std::getenv("GFQ_PROF_DUMP_TASKS"))
        for (auto& r : recs) {
          float t = 0, t0 = 0;
          if (cudaEventElapsedTime(&t, r.e0, r.e1) == cudaSuccess &&
              cudaEventElapsedTime(&t0, recs.front().e0, r.e0) == cudaSuccess)
            std::fprintf(fh, "T %d %.4f %.4f %.1f %s\n", r.path, double(t0), double(t0) + double(t), r.ops,
                         r.task ? r.task : "-");
        }
      std::fclose(fh);
    }
  }
  for (auto& r : recs) {
    cudaEventDestroy(r.e0);
    cudaEventDestroy(r.e1);
  }
  cudaGetLastError();
  if (union_ms)
    for (int q = 0; q < n; ++q) {
      auto& v = iv[std::size_t(q)];
      std::sort(v.begin(), v.end());
      double tot = 0, lo = 0, hi = -1e300;
      for (const auto& [a, b] : v) {
        if (a > hi) {
          if (hi > lo) tot += hi - lo;
          lo = a;
          hi = b;
        } else if (b > hi) {
          hi = b;
        }
      }
      if (hi > lo) tot += hi - lo;
      union_ms[q] = tot;
    }
}

void profile_take(std::int64_t launches[2], double ops[2], double ms[2]) {
  profile_take_kinds(2, launches, ops, ms, nullptr);
}

void set_mad_policy(int policy) { g_policy = policy; }
// K1f dispatch: small fields, tiles that fill the 128 x 192 grid, and
// enough work that the two packing passes (1.5 B per operand element) stay
// small next to the contraction; GFQ_NO_F4 keeps every product on kind::i8.
// Streams at the device's greatest priority carry the Step-1 critical path
// (the executor's ClearDown / UpdateRow(i, j, j+1) stream).
bool stream_is_critical(cudaStream_t s) {
  static const int greatest = [] {
    int lo = 0, hi = 0;
    GFQ_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    return hi;
  }();
  if (s == nullptr) return false;
  int pr = 0;
  if (cudaStreamGetPriority(s, &pr) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return pr == greatest && greatest != 0;
}
namespace {
// GFQ_PARTITION=1 also turns it on outside the Chief (job-level experiments)
std::atomic<bool> g_partition{[] {
  const char* e = std::getenv("GFQ_PARTITION");
  return e && e[0] == '1';
}()};
}  // namespace
void set_critical_partition(bool on) { g_partition = on; }
bool critical_partition() { return g_partition; }
namespace {
// Steps 2-3 (the back substitution) run after the last ClearDown: no
// critical path is left to keep SMs free for
bool late_task() {
  const char* t = hprof::t_task_name;
  return std::strncmp(t, "ClearUp", 7) == 0 || std::strncmp(t, "PreClearUp", 10) == 0;
}
}  // namespace
int k1_sms(cudaStream_t s) {
  static const int reserve = [] {
    const char* e = std::getenv("GFQ_K1_SM_RESERVE");
    return e ? std::atoi(e) : 16;
  }();
  static const int crit = [] {
    const char* e = std::getenv("GFQ_CRIT_GRID");
    return e ? std::atoi(e) : 0;
  }();
  if (stream_is_critical(s))
    return crit > 0 && std::strcmp(hprof::t_task_name, "ClearDown") == 0 ? std::min(crit, sm_count()) : sm_count();
  static const bool late_reserve = std::getenv("GFQ_LATE_RESERVE") != nullptr;  // A/B
  if (reserve <= 0 || !g_partition || (late_task() && !late_reserve)) return sm_count();
  return std::max(1, sm_count() - reserve);
}
// The K1 lane (GFQ_K1_LANE=1): persistent contractions issued from
// non-critical streams run one at a time (each waits for the previous one
// on any stream), so together with GFQ_K1_SM_RESERVE they never occupy the
// reserved SMs the critical path's kernels need.
namespace {
std::mutex g_lane_mtx;
cudaEvent_t g_lane_ev[64];
int g_lane_n = 0;
bool g_lane_has = false;
}  // namespace
K1Lane::K1Lane(cudaStream_t s) : s_(s) {
  static const bool on = [] {
    const char* e = std::getenv("GFQ_K1_LANE");
    return !(e && e[0] == '0');
  }();
  static const bool late_lane = std::getenv("GFQ_LATE_LANE") != nullptr;  // A/B
  if (!on || !g_partition || stream_is_critical(s) || (late_task() && !late_lane)) return;
  g_lane_mtx.lock();
  held_ = true;
  if (!g_lane_n) {
    for (auto& e : g_lane_ev) GFQ_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    g_lane_n = 64;
  }
  static int cur = 0;
  if (g_lane_has) GFQ_CUDA(cudaStreamWaitEvent(s, g_lane_ev[cur], 0));
  cur_ = &cur;
}
K1Lane::~K1Lane() {
  if (!held_) return;
  *cur_ = (*cur_ + 1) % g_lane_n;
  cudaEventRecord(g_lane_ev[*cur_], s_);
  g_lane_has = true;
  g_lane_mtx.unlock();
}
bool use_f4(std::uint32_t p, std::int64_t m, std::int64_t n, std::int64_t k) {
  static const bool off = std::getenv("GFQ_NO_F4") != nullptr;
  static const double min_work = [] {
    const char* e = std::getenv("GFQ_F4_MIN_MACS");
    return e ? std::atof(e) : 1.0e11;
  }();
  const int pol = g_policy;
  if (!f4_field(p) || pol == 1 || pol == 2 || m <= 0 || n <= 0 || k <= 0) return false;
  if (pol == 3) return true;
  if (off) return false;
  return m >= 128 && n >= 192 && k >= 128 && double(m) * double(n) * double(k) >= min_work;
}
int mad_policy() { return g_policy; }
void mad_counters(std::int64_t* simt, std::int64_t* tc) {
  *simt = g_simt;
  *tc = g_tc;
}
void reset_mad_counters() {
  g_simt = 0;
  g_tc = 0;
}

void mad(std::uint32_t p, std::int64_t m, std::int64_t n, std::int64_t k,
         const std::uint8_t* A, std::int64_t lda, const std::uint8_t* B,
         std::int64_t ldb, const std::uint8_t* Cin, std::int64_t ldc,
         std::uint8_t* D, std::int64_t ldd, cudaStream_t s) {
  if (m == 0 || n == 0) return;
  hprof::Scope hp(hprof::kMad);
  const int pol = g_policy;
  // The tcgen05 path pays a prologue (TMEM alloc, barrier init, descriptor
  // fetch) of a few microseconds; below ~4 Mi MACs or for K < 32 (one MMA
  // instruction) the SIMT kernel is as fast and exactly as exact.
  // Deep-K skinny products (e.g. n = 1 when a block column has one
  // remaining non-pivot column) also belong on K1: the SIMT tile kernel
  // would stream K through 64-wide tiles with a tiny grid.
  const bool big = k >= 32 && (double(m) * double(n) * double(k) >= 4.0 * 1024 * 1024 || k >= 128);
  const bool prof = g_profile;
  ProfRec rec{nullptr, nullptr, 2.0 * double(m) * double(n) * double(k), 0, hprof::t_task_name};
  if (prof) {
    GFQ_CUDA(cudaEventCreate(&rec.e0));
    GFQ_CUDA(cudaEventCreate(&rec.e1));
    GFQ_CUDA(cudaEventRecord(rec.e0, s));
  }
  bool done = false;
  const auto al = [](const void* q, std::int64_t ld) {
    return q == nullptr || ((reinterpret_cast<std::uintptr_t>(q) & 15) == 0 && (ld & 15) == 0);
  };
  if (pol != 2 && k >= 1 && k <= kSmallK && al(B, ldb) && al(Cin, ldc) && al(D, ldd)) {
    ++g_simt;
    rec.path = 1;
    const std::int64_t total = m * ((n + 15) / 16);
    const std::int64_t cap = std::int64_t(sm_count()) * 8;
    const unsigned grid = unsigned(std::min<std::int64_t>((total + 255) / 256, cap));
    GFQ_CUDA(launch_pdl(mad_smallk_kernel<false>, dim3(grid), dim3(256), 0, s, p, magic_of(p), int(m), int(n), int(k), A, lda, B, ldb,
                                           Cin, ldc, D, ldd, SmallkMaps{nullptr, nullptr, nullptr}));
    GFQ_CUDA(cudaGetLastError());
    count_launch();
    done = true;
  }
  if (!done && pol != 1 && k > 0 && (pol == 2 || big)) {
    if (mad_tc(p, m, n, k, A, lda, B, ldb, Cin, ldc, D, ldd, s)) {
      ++g_tc;
      done = true;
    }
  }
  if (!done) {
    ++g_simt;
    rec.path = 1;
    mad_simt(p, m, n, k, A, lda, B, ldb, Cin, ldc, D, ldd, s);
  }
  if (prof) {
    GFQ_CUDA(cudaEventRecord(rec.e1, s));
    std::lock_guard<std::mutex> lk(g_prof_mtx);
    g_prof.push_back(rec);
  }
  // developer log of every contraction's shape and path (GFQ_MAD_LOG)
  static const bool log = std::getenv("GFQ_MAD_LOG") != nullptr;
  if (log)
    std::fprintf(stderr, "mad m=%lld n=%lld k=%lld path=%s task=%s\n", static_cast<long long>(m),
                 static_cast<long long>(n), static_cast<long long>(k), rec.path ? "simt" : "tc", hprof::t_task_name);
}

void mad_smallk_maps(std::uint32_t p, std::int64_t m, std::int64_t n, std::int64_t k,
                     const std::uint8_t* A, std::int64_t lda, const std::uint8_t* B, std::int64_t ldb,
                     const std::int32_t* brm, const std::uint8_t* Cin, std::int64_t ldc,
                     const std::int32_t* crm, std::uint8_t* D, std::int64_t ldd, const std::int32_t* drm,
                     cudaStream_t s) {
  if (m == 0 || n == 0) return;
  if (k < 1 || k > kSmallK) throw std::invalid_argument("mad_smallk_maps: k must be 1..32");
  const auto al = [](const void* q, std::int64_t ld) {
    return q == nullptr || ((reinterpret_cast<std::uintptr_t>(q) & 15) == 0 && (ld & 15) == 0);
  };
  if (!al(B, ldb) || !al(Cin, ldc) || !al(D, ldd))
    throw std::invalid_argument("mad_smallk_maps: operands must be 16-byte aligned");
  hprof::Scope hp(hprof::kMad);
  ProfScope ps(kProfSimt, 2.0 * double(m) * double(n) * double(k), s);
  const std::int64_t total = m * ((n + 15) / 16);
  const std::int64_t cap = std::int64_t(sm_count()) * 8;
  const unsigned grid = unsigned(std::min<std::int64_t>((total + 255) / 256, cap));
  GFQ_CUDA(launch_pdl(mad_smallk_kernel<true>, dim3(grid), dim3(256), 0, s, p, magic_of(p), int(m), int(n),
                      int(k), A, lda, B, ldb, Cin, ldc, D, ldd, SmallkMaps{brm, crm, drm}));
  count_launch();
}

// ------------------------------------------------------------------ K3/K4
namespace {
__device__ __forceinline__ const std::uint8_t* pick_row(
    const std::uint8_t* A, std::int64_t lda, const std::uint8_t* B,
    std::int64_t ldb, const std::int32_t* rmap, std::int64_t i, bool& fromB) {
  if (!rmap) {
    fromB = false;
    return A + i * lda;
  }
  const std::int32_t v = rmap[i];
  if (v == -1) return nullptr;
  if (v >= 0) {
    fromB = false;
    return A + std::int64_t(v) * lda;
  }
  fromB = true;
  return B + std::int64_t(-v - 2) * ldb;
}

// Row-only select, 16-byte vectorised (all pointers/strides 16B-aligned).
__global__ void select_rows_v16_kernel(std::uint8_t* dst, std::int64_t ldd,
                                       std::int64_t rows, std::int64_t cols,
                                       const std::uint8_t* A, std::int64_t lda,
                                       const std::uint8_t* B, std::int64_t ldb,
                                       const std::int32_t* rmap) {
  pdl_wait_and_release();
  const std::int64_t nvec = (cols + 15) / 16;
  for (std::int64_t i = blockIdx.y; i < rows; i += gridDim.y) {
    bool fromB = false;
    const std::uint8_t* src = pick_row(A, lda, B, ldb, rmap, i, fromB);
    uint4* drow = reinterpret_cast<uint4*>(dst + i * ldd);
    for (std::int64_t v = blockIdx.x * blockDim.x + threadIdx.x; v < nvec;
         v += std::int64_t(gridDim.x) * blockDim.x) {
      if (v * 16 + 16 <= cols) {
        drow[v] = src ? reinterpret_cast<const uint4*>(src)[v] : make_uint4(0, 0, 0, 0);
      } else {
        for (std::int64_t c = v * 16; c < cols; ++c)
          dst[i * ldd + c] = src ? src[c] : 0;
      }
    }
  }
}

__global__ void select2d_kernel(std::uint8_t* dst, std::int64_t ldd,
                                std::int64_t rows, std::int64_t cols,
                                const std::uint8_t* A, std::int64_t lda,
                                const std::uint8_t* B, std::int64_t ldb,
                                const std::int32_t* rmap,
                                const std::int32_t* cmap) {
  pdl_wait_and_release();
  for (std::int64_t i = blockIdx.y; i < rows; i += gridDim.y) {
    std::int32_t rv = -3;  // "no row map"
    if (rmap) rv = rmap[i];
    for (std::int64_t j = blockIdx.x * blockDim.x + threadIdx.x; j < cols;
         j += std::int64_t(gridDim.x) * blockDim.x) {
      std::uint8_t out = 0;
      const std::int32_t cv = cmap ? cmap[j] : std::int32_t(j);
      if (rv != -1 && cv != -1) {
        const bool rowB = rmap && rv <= -2;
        const bool colB = cmap && cv <= -2;
        const std::int64_t r = rmap ? (rowB ? -rv - 2 : rv) : i;
        const std::int64_t c = colB ? -cv - 2 : cv;
        out = (rowB || colB) ? B[r * ldb + c] : A[r * lda + c];
      }
      dst[i * ldd + j] = out;
    }
  }
}

// General select (column map present), 16 output columns per thread and
// kSelRows rows per block: the 16 column-map entries are read (as int4
// vectors) and classified once, then reused for every row of the block's
// row group -- the map costs 64 B of loads per 16 B of payload otherwise.
// A contiguous run of one source row (crz / RowLengthen: long runs with a
// few inserted zero columns) takes two aligned 16-byte loads and funnel
// shifts; anything else 16 byte loads.  16-byte stores (dst rows 16B-aligned).
constexpr int kSelRows = 8;
__global__ void select2d_v16_kernel(std::uint8_t* dst, std::int64_t ldd,
                                    std::int64_t rows, std::int64_t cols,
                                    const std::uint8_t* A, std::int64_t lda,
                                    const std::uint8_t* B, std::int64_t ldb,
                                    const std::int32_t* rmap,
                                    const std::int32_t* cmap) {
  pdl_wait_and_release();
  const std::int64_t nvec = (cols + 15) / 16;
  for (std::int64_t v = blockIdx.x * blockDim.x + threadIdx.x; v < nvec;
       v += std::int64_t(gridDim.x) * blockDim.x) {
    const std::int64_t j0 = v * 16;
    std::int32_t cm[16];
    if (j0 + 16 <= cols && (reinterpret_cast<std::uintptr_t>(cmap + j0) & 15) == 0) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int4 c4 = reinterpret_cast<const int4*>(cmap + j0)[q];
        cm[4 * q] = c4.x;
        cm[4 * q + 1] = c4.y;
        cm[4 * q + 2] = c4.z;
        cm[4 * q + 3] = c4.w;
      }
    } else {
#pragma unroll
      for (int q = 0; q < 16; ++q) cm[q] = j0 + q < cols ? cmap[j0 + q] : -1;
    }
    const std::int32_t c0 = cm[0];
    bool run = c0 != -1;
#pragma unroll
    for (int q = 1; q < 16; ++q) run = run && (c0 >= 0 ? cm[q] == c0 + q : cm[q] == c0 - q);
    bool zero = true;
#pragma unroll
    for (int q = 0; q < 16; ++q) zero = zero && cm[q] == -1;
    const bool colB = c0 <= -2;                       // the run's source operand
    const std::int64_t sc = c0 >= 0 ? c0 : std::int64_t(-c0 - 2);
    for (std::int64_t i0 = std::int64_t(blockIdx.y) * kSelRows; i0 < rows;
         i0 += std::int64_t(gridDim.y) * kSelRows) {
      const std::int64_t i1 = i0 + kSelRows < rows ? i0 + kSelRows : rows;
      for (std::int64_t i = i0; i < i1; ++i) {
        std::int32_t rv = -3;  // "no row map"
        if (rmap) rv = rmap[i];
        const bool rowB = rmap && rv <= -2;
        const std::int64_t r = rmap ? (rowB ? -rv - 2 : rv) : i;
        const std::uint8_t* arow = (rv == -1 || rowB) ? nullptr : A + r * lda;
        const std::uint8_t* brow = B ? B + (rowB ? r : (rmap ? r : i)) * ldb : nullptr;
        std::uint32_t w[4] = {0, 0, 0, 0};
        if (rv != -1 && !zero) {
          const std::uint8_t* srow = colB ? brow : (rowB ? brow : arow);
          const std::int64_t sld = (colB || rowB) ? ldb : lda;
          if (run && srow && ((reinterpret_cast<std::uintptr_t>(srow) | std::uintptr_t(sld)) & 15) == 0 &&
              (sc & ~std::int64_t(15)) + 32 <= sld) {
            const uint4* p16 = reinterpret_cast<const uint4*>(srow + (sc & ~std::int64_t(15)));
            const uint4 lo = p16[0];
            const int sh = int(sc & 15);
            if (sh == 0) {
              w[0] = lo.x; w[1] = lo.y; w[2] = lo.z; w[3] = lo.w;
            } else {
              const uint4 hi = p16[1];
              std::uint32_t u[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
              const int wq = sh >> 2, bs = 8 * (sh & 3);
              // word shift by wq in two register-resident stages (no dynamic
              // indexing, which would spill the array to local memory)
#pragma unroll
              for (int q = 0; q < 6; ++q) u[q] = (wq & 2) ? u[q + 2] : u[q];
#pragma unroll
              for (int q = 0; q < 5; ++q) u[q] = (wq & 1) ? u[q + 1] : u[q];
#pragma unroll
              for (int q = 0; q < 4; ++q) w[q] = bs ? __funnelshift_r(u[q], u[q + 1], bs) : u[q];
            }
          } else {
#pragma unroll
            for (int q = 0; q < 16; ++q) {
              const std::int32_t cv = cm[q];
              std::uint32_t x = 0;
              if (cv >= 0) {
                x = rowB ? brow[cv] : arow[cv];
              } else if (cv <= -2) {
                x = brow[-cv - 2];
              }
              w[q >> 2] |= x << (8 * (q & 3));
            }
          }
        }
        if (j0 + 16 <= cols) {
          *reinterpret_cast<uint4*>(dst + i * ldd + j0) = make_uint4(w[0], w[1], w[2], w[3]);
        } else {
          for (std::int64_t c = j0; c < cols; ++c)
            dst[i * ldd + c] = std::uint8_t((w[(c - j0) >> 2] >> (8 * ((c - j0) & 3))) & 0xFF);
        }
      }
    }
  }
}

__global__ void set_entries_kernel(std::uint8_t* dst, std::int64_t ldd,
                                   const std::int32_t* pos, std::int64_t n,
                                   std::uint8_t value) {
  pdl_wait_and_release();
  for (std::int64_t q = blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += std::int64_t(gridDim.x) * blockDim.x)
    dst[std::int64_t(pos[2 * q]) * ldd + pos[2 * q + 1]] = value;
}
}  // namespace

namespace {
// select2d with the row / column maps passed IN the launch parameters
// (int16 entries: rows first, then columns): no upload, so no extra CUDA
// call on the host.  A block handles up to 2048 output columns (16 a thread)
// for a strided set of rows; the column map is staged once per block in
// shared memory, the row map is read uniformly per row.
template <int CAP>
__global__ void __launch_bounds__(128)
select_inline_kernel(std::uint8_t* dst, std::int64_t ldd, std::int64_t rows, std::int64_t cols,
                     const std::uint8_t* A, std::int64_t lda, const std::uint8_t* B,
                     std::int64_t ldb, const __grid_constant__ InlineMaps<CAP> maps) {
  pdl_wait_and_release();
  __shared__ std::int32_t scm[2048];
  const std::int64_t nr = maps.nr, nc = maps.nc;
  const std::int64_t c0 = std::int64_t(blockIdx.x) * 2048;
  const std::int64_t cn = cols - c0 < 2048 ? cols - c0 : 2048;
  if (nc)
    for (int e = threadIdx.x; e < cn; e += blockDim.x) scm[e] = maps.v[nr + c0 + e];
  __syncthreads();
  const std::int64_t j0 = c0 + 16 * threadIdx.x;
  if (j0 >= cols) return;
  const bool full = j0 + 16 <= cols;
  for (std::int64_t i = blockIdx.y; i < rows; i += gridDim.y) {
    const std::int32_t rv = nr ? maps.v[i] : std::int32_t(i);
    const bool rowB = nr && rv <= -2;
    const std::int64_t r = rowB ? -rv - 2 : rv;
    const std::uint8_t* arow = (rv == -1 || rowB) ? nullptr : A + r * lda;
    const std::uint8_t* brow = B ? B + (rowB ? r : (nr ? r : i)) * ldb : nullptr;
    std::uint32_t w[4] = {0, 0, 0, 0};
    if (rv != -1) {
      if (!nc) {
        const std::uint8_t* src = rowB ? brow : arow;
        if (full) {
          const uint4 x = *reinterpret_cast<const uint4*>(src + j0);
          w[0] = x.x; w[1] = x.y; w[2] = x.z; w[3] = x.w;
        } else {
          for (int q = 0; q < 16; ++q)
            if (j0 + q < cols) w[q >> 2] |= std::uint32_t(src[j0 + q]) << (8 * (q & 3));
        }
      } else {
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          if (j0 + q >= cols) break;
          const std::int32_t cv = scm[16 * threadIdx.x + q];
          std::uint32_t x = 0;
          if (cv >= 0) x = rowB ? brow[cv] : arow[cv];
          else if (cv <= -2) x = brow[-cv - 2];
          w[q >> 2] |= x << (8 * (q & 3));
        }
      }
    }
    std::uint8_t* drow = dst + i * ldd + j0;
    if (full) {
      *reinterpret_cast<uint4*>(drow) = make_uint4(w[0], w[1], w[2], w[3]);
    } else {
      for (std::int64_t c = 0; c < cols - j0; ++c) drow[c] = std::uint8_t((w[c >> 2] >> (8 * (c & 3))) & 0xFF);
    }
  }
}

template <int CAP>
bool launch_inline(std::uint8_t* dst, std::int64_t ldd, std::int64_t rows, std::int64_t cols,
                   const std::uint8_t* A, std::int64_t lda, const std::uint8_t* B, std::int64_t ldb,
                   const std::int32_t* rmap, const std::int32_t* cmap, cudaStream_t s) {
  InlineMaps<CAP> m;
  m.nr = rmap ? std::int32_t(rows) : 0;
  m.nc = cmap ? std::int32_t(cols) : 0;
  for (std::int64_t i = 0; i < m.nr; ++i) m.v[i] = std::int16_t(rmap[i]);
  for (std::int64_t j = 0; j < m.nc; ++j) m.v[m.nr + j] = std::int16_t(cmap[j]);
  const unsigned gx = unsigned((cols + 2047) / 2048);
  const unsigned gy = unsigned(rows < 256 ? rows : 256);
  GFQ_CUDA(launch_pdl(select_inline_kernel<CAP>, dim3(dim3(gx, gy)), dim3(128), 0, s, dst, ldd, rows, cols, A, lda, B, ldb, m));
  GFQ_CUDA(cudaGetLastError());
  count_launch();
  return true;
}
}  // namespace

bool select2d_inline(std::uint8_t* dst, std::int64_t ldd, std::int64_t rows, std::int64_t cols,
                     const std::uint8_t* A, std::int64_t lda, const std::uint8_t* B,
                     std::int64_t ldb, const std::int32_t* rmap, const std::int32_t* cmap,
                     cudaStream_t s) {
  if (rows == 0 || cols == 0) return true;
  const std::int64_t n = (rmap ? rows : 0) + (cmap ? cols : 0);
  const auto al = [](const void* ptr, std::int64_t ld) {
    return ptr == nullptr || ((reinterpret_cast<std::uintptr_t>(ptr) & 15) == 0 && (ld & 15) == 0);
  };
  // large gathers take the upload path: the upload is cheap next to them and
  // the regular kernels spread rows over far more blocks
  if (n > 4096 || !al(dst, ldd) || rows * cols > (std::int64_t(1) << 20) ||
      (!cmap && !(al(A, lda) && al(B, ldb))))
    return false;
  const auto fits = [](const std::int32_t* m, std::int64_t k) {
    for (std::int64_t i = 0; i < k; ++i)
      if (m[i] < -32768 || m[i] > 32767) return false;
    return true;
  };
  if ((rmap && !fits(rmap, rows)) || (cmap && !fits(cmap, cols))) return false;
  hprof::Scope hp(hprof::kSelect);
  static const bool log = std::getenv("GFQ_MAD_LOG") != nullptr;
  if (log)
    std::fprintf(stderr, "select rows=%lld cols=%lld rmap=%d cmap=%d task=%s inline\n", static_cast<long long>(rows),
                 static_cast<long long>(cols), rmap ? 1 : 0, cmap ? 1 : 0, hprof::t_task_name);
  ProfScope ps(kProfSelect, 2.0 * double(rows) * double(cols) + 4.0 * double(n), s);
  if (n <= 512) return launch_inline<512>(dst, ldd, rows, cols, A, lda, B, ldb, rmap, cmap, s);
  if (n <= 1536) return launch_inline<1536>(dst, ldd, rows, cols, A, lda, B, ldb, rmap, cmap, s);
  return launch_inline<4096>(dst, ldd, rows, cols, A, lda, B, ldb, rmap, cmap, s);
}

void select2d(std::uint8_t* dst, std::int64_t ldd, std::int64_t rows,
              std::int64_t cols, const std::uint8_t* A, std::int64_t lda,
              const std::uint8_t* B, std::int64_t ldb, const std::int32_t* rmap,
              const std::int32_t* cmap, cudaStream_t s) {
  if (rows == 0 || cols == 0) return;
  hprof::Scope hp(hprof::kSelect);
  static const bool log = std::getenv("GFQ_MAD_LOG") != nullptr;
  if (log)
    std::fprintf(stderr, "select rows=%lld cols=%lld rmap=%d cmap=%d task=%s\n", static_cast<long long>(rows),
                 static_cast<long long>(cols), rmap ? 1 : 0, cmap ? 1 : 0, hprof::t_task_name);
  ProfScope ps(kProfSelect,
               2.0 * double(rows) * double(cols) + 4.0 * double((rmap ? rows : 0) + (cmap ? cols : 0)), s);
  const unsigned gy = unsigned(rows < 65535 ? rows : 65535);
  const auto al = [](const void* ptr, std::int64_t ld) {
    return ptr == nullptr ||
           ((reinterpret_cast<std::uintptr_t>(ptr) & 15) == 0 && (ld & 15) == 0);
  };
  if (!cmap && al(dst, ldd) && al(A, lda) && al(B, ldb)) {
    const std::int64_t nvec = (cols + 15) / 16;
    const unsigned gx = unsigned((nvec + 127) / 128);
    GFQ_CUDA(launch_pdl(select_rows_v16_kernel, dim3(dim3(gx, gy)), dim3(128), 0, s, dst, ldd, rows, cols, A, lda, B, ldb, rmap));
  } else if (cmap && al(dst, ldd)) {
    const std::int64_t nvec = (cols + 15) / 16;
    const unsigned gx = unsigned((nvec + 127) / 128);
    const std::int64_t ry = (rows + kSelRows - 1) / kSelRows;
    const unsigned gyr = unsigned(ry < 65535 ? ry : 65535);
    GFQ_CUDA(launch_pdl(select2d_v16_kernel, dim3(dim3(gx, gyr)), dim3(128), 0, s, dst, ldd, rows, cols, A, lda, B, ldb, rmap, cmap));
  } else {
    const unsigned gx = unsigned((cols + 255) / 256);
    GFQ_CUDA(launch_pdl(select2d_kernel, dim3(dim3(gx, gy)), dim3(256), 0, s, dst, ldd, rows, cols, A, lda, B, ldb, rmap, cmap));
  }
  GFQ_CUDA(cudaGetLastError());
    count_launch();
}

namespace {
// dst rows [0, rows) x bytes [0, width) = value (16-byte stores where aligned)
__global__ void fill2d_kernel(std::uint8_t* dst, std::int64_t ldd, std::int64_t rows, std::int64_t width,
                              std::uint8_t value) {
  pdl_wait_and_release();
  const std::uint32_t v4 = 0x01010101u * value;
  const bool al = ((reinterpret_cast<std::uintptr_t>(dst) | std::uintptr_t(ldd)) & 15) == 0;
  const std::int64_t nv = al ? width / 16 : 0;
  for (std::int64_t i = blockIdx.y; i < rows; i += gridDim.y) {
    std::uint8_t* row = dst + i * ldd;
    for (std::int64_t v = std::int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < nv;
         v += std::int64_t(gridDim.x) * blockDim.x)
      reinterpret_cast<uint4*>(row)[v] = make_uint4(v4, v4, v4, v4);
    for (std::int64_t b = nv * 16 + std::int64_t(blockIdx.x) * blockDim.x + threadIdx.x; b < width;
         b += std::int64_t(gridDim.x) * blockDim.x)
      row[b] = value;
  }
}
__global__ void copy_from_mapped_kernel(std::uint8_t* dst, const std::uint8_t* src, std::size_t bytes) {
  pdl_wait_and_release();
  const std::size_t nv = bytes / 16;
  for (std::size_t v = std::size_t(blockIdx.x) * blockDim.x + threadIdx.x; v < nv;
       v += std::size_t(gridDim.x) * blockDim.x)
    // .cv loads: a ring slot is rewritten by the host between uploads, so no
    // cached copy of an earlier content may be used
    reinterpret_cast<uint4*>(dst)[v] = __ldcv(reinterpret_cast<const uint4*>(src) + v);
  for (std::size_t b = nv * 16 + 4 * (std::size_t(blockIdx.x) * blockDim.x + threadIdx.x); b < bytes;
       b += 4 * std::size_t(gridDim.x) * blockDim.x)
    *reinterpret_cast<std::uint32_t*>(dst + b) = __ldcv(reinterpret_cast<const unsigned int*>(src + b));
}
}  // namespace

void fill2d(std::uint8_t* dst, std::int64_t ldd, std::int64_t rows, std::int64_t width, std::uint8_t value,
            cudaStream_t s) {
  if (rows <= 0 || width <= 0) return;
  const std::int64_t per_row = (width + 15) / 16;
  const unsigned gx = unsigned(std::min<std::int64_t>((per_row + 255) / 256, 64));
  const unsigned gy = unsigned(std::min<std::int64_t>(rows, 65535));
  GFQ_CUDA(launch_pdl(fill2d_kernel, dim3(gx, gy), dim3(256), 0, s, dst, ldd, rows, width, value));
  count_launch();
}

namespace {
__global__ void copy_to_mapped_kernel(std::uint8_t* dst, const std::uint8_t* src, std::size_t bytes) {
  pdl_wait_and_release();
  for (std::size_t b = 4 * (std::size_t(blockIdx.x) * blockDim.x + threadIdx.x); b < bytes;
       b += 4 * std::size_t(gridDim.x) * blockDim.x)
    __stcs(reinterpret_cast<unsigned int*>(dst + b), *reinterpret_cast<const unsigned int*>(src + b));
}
}  // namespace

void copy_to_mapped(std::uint8_t* dst, const std::uint8_t* src, std::size_t bytes, cudaStream_t s) {
  if (bytes == 0) return;
  const unsigned grid = unsigned(std::min<std::size_t>((bytes / 4 + 255) / 256, 32));
  GFQ_CUDA(launch_pdl(copy_to_mapped_kernel, dim3(grid), dim3(256), 0, s, dst, src, bytes));
  count_launch();
}

void copy_from_mapped(std::uint8_t* dst, const std::uint8_t* src, std::size_t bytes, cudaStream_t s) {
  if (bytes == 0) return;
  const std::size_t nv = (bytes + 15) / 16;
  const unsigned grid = unsigned(std::min<std::size_t>((nv + 255) / 256, 64));
  GFQ_CUDA(launch_pdl(copy_from_mapped_kernel, dim3(grid), dim3(256), 0, s, dst, src, bytes));
  count_launch();
}

void set_entries(std::uint8_t* dst, std::int64_t ldd, const std::int32_t* pos,
                 std::int64_t n, std::uint8_t value, cudaStream_t s) {
  if (n == 0) return;
  GFQ_CUDA(launch_pdl(set_entries_kernel, dim3(unsigned((n + 255) / 256)), dim3(256), 0, s, dst, ldd, pos, n, value));
  GFQ_CUDA(cudaGetLastError());
    count_launch();
}

// ------------------------------------------------------------------ K2 base
namespace {
__device__ __forceinline__ std::uint32_t powmod(std::uint32_t a, std::uint32_t e,
                                                std::uint32_t p) {
  std::uint32_t r = 1, b = a % p;
  while (e) {
    if (e & 1) r = (r * b) % p;
    b = (b * b) % p;
    e >>= 1;
  }
  return r;
}

// One CTA.  Shared layout: w[rows][cols] | t[rows][rmax] | coef[rows] |
// piv[rows] | inv[256].  Column-wise Gauss-Jordan, pivot = first
// non-pivotal row with a nonzero entry (reference src/chief.cpp:436-460;
// equivalent to direct_gauss's row-wise rule).
__global__ void __launch_bounds__(1024)
ech_base_kernel(std::uint32_t p, std::uint32_t magic, int rows, int cols,
                const std::uint8_t* __restrict__ H, std::int64_t ldh,
                std::uint8_t* W, std::int64_t ldw, std::uint8_t* Tc,
                std::int64_t ldt, std::int32_t* info) {
  extern __shared__ __align__(16) std::uint8_t sm[];
  const int rmax = rows < cols ? rows : cols;
  std::uint8_t* w = sm;
  std::uint8_t* t = w + rows * cols;
  std::uint8_t* coef = t + rows * (rmax > 0 ? rmax : 1);
  std::uint8_t* piv = coef + rows;
  std::uint8_t* invt = piv + rows;
  __shared__ int sel_s;
  __shared__ int pcol[kEchBaseMax], prow[kEchBaseMax];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;

  for (int e = tid; e < rows * cols; e += nt)
    w[e] = H[std::int64_t(e / cols) * ldh + (e % cols)];
  for (int e = tid; e < rows * rmax; e += nt) t[e] = 0;
  for (int e = tid; e < rows; e += nt) piv[e] = 0;
  for (int a = tid; a < 256; a += nt)
    invt[a] = (a > 0 && std::uint32_t(a) < p) ? std::uint8_t(powmod(a, p - 2, p)) : 0;
  __syncthreads();

  int r = 0;
  __shared__ int sel_c;
  for (int col = 0; col < cols && r < rmax; ++col) {
    if (cols > rows) {
      // short-wide blocks: jump to the next column holding a nonzero in a
      // non-pivotal row (O(rows x cols) a pivot instead of a barrier round
      // per column)
      if (tid == 0) sel_c = cols;
      __syncthreads();
      const int span = cols - col;
      for (int e = tid; e < rows * span; e += nt) {
        const int i = e / span, c = col + e % span;
        if (!piv[i] && w[i * cols + c]) atomicMin(&sel_c, c);
      }
      __syncthreads();
      col = sel_c;
      if (col == cols) break;  // block-uniform
    }
    if (tid == 0) sel_s = rows;
    __syncthreads();
    for (int i = tid; i < rows; i += nt)
      if (!piv[i] && w[i * cols + col]) atomicMin(&sel_s, i);
    __syncthreads();
    const int s = sel_s;
    if (s == rows) continue;  // block-uniform
    const std::uint32_t scale = p - invt[w[s * cols + col]];
    for (int i = tid; i < rows; i += nt) coef[i] = (i == s) ? 0 : w[i * cols + col];
    __syncthreads();
    // normalise the pivot row: pivot entry becomes -1
    const int wcols = cols - col;
    for (int c = tid; c < wcols; c += nt)
      w[s * cols + col + c] = std::uint8_t(modp(scale * w[s * cols + col + c], p, magic));
    for (int q = tid; q <= r; q += nt)
      t[s * rmax + q] = q == r ? std::uint8_t(scale)
                               : std::uint8_t(modp(scale * t[s * rmax + q], p, magic));
    __syncthreads();
    // eliminate column `col` from every other row (Gauss-Jordan)
    const int width = wcols + r + 1;
    for (int i = warp; i < rows; i += nw) {
      const std::uint32_t cf = coef[i];
      if (!cf) continue;
      for (int e = lane; e < width; e += 32) {
        if (e < wcols) {
          const int idx = i * cols + col + e;
          const std::uint32_t b = w[s * cols + col + e];
          w[idx] = p == 2 ? std::uint8_t(w[idx] ^ b)
                          : std::uint8_t(modp(w[idx] + cf * b, p, magic));
        } else {
          const int q = e - wcols;
          const int idx = i * rmax + q;
          const std::uint32_t b = t[s * rmax + q];
          t[idx] = p == 2 ? std::uint8_t(t[idx] ^ b)
                          : std::uint8_t(modp(t[idx] + cf * b, p, magic));
        }
      }
    }
    if (tid == 0) {
      piv[s] = 1;
      pcol[r] = col;
      prow[r] = s;
    }
    ++r;
    __syncthreads();
  }
  for (int e = tid; e < rows * cols; e += nt)
    W[std::int64_t(e / cols) * ldw + (e % cols)] = w[e];
  if (r > 0)
    for (int e = tid; e < rows * r; e += nt)
      Tc[std::int64_t(e / r) * ldt + (e % r)] = t[(e / r) * rmax + (e % r)];
  if (tid == 0) info[0] = r;
  for (int q = tid; q < r; q += nt) {
    info[1 + q] = pcol[q];
    info[1 + rmax + q] = prow[q];
  }
}
}  // namespace

std::size_t ech_base_smem(std::int64_t rows, std::int64_t cols) {
  const std::int64_t rmax = rows < cols ? rows : cols;
  return std::size_t(rows * cols + rows * (rmax > 0 ? rmax : 1) + 2 * rows + 256);
}
bool ech_base_fits(std::int64_t rows, std::int64_t cols) {
  const std::int64_t rmax = rows < cols ? rows : cols;
  return rmax <= kEchBaseMax && ech_base_smem(rows, cols) <= kEchBaseSmem &&
         (rmax <= kEchThinMax || (rows <= kEchBaseMax && cols <= kEchBaseMax));
}

void ech_base(std::uint32_t p, std::int64_t rows, std::int64_t cols,
              const std::uint8_t* H, std::int64_t ldh, std::uint8_t* W,
              std::int64_t ldw, std::uint8_t* Tc, std::int64_t ldt,
              std::int32_t* info, cudaStream_t s) {
  if (!ech_base_fits(rows, cols)) throw std::invalid_argument("ech_base: block exceeds the base-case size");
  const std::size_t smem = ech_base_smem(rows, cols);
  static bool attr_set = false;
  if (!attr_set) {
    GFQ_CUDA(cudaFuncSetAttribute(ech_base_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(kEchBaseSmem)));
    attr_set = true;
  }
  int threads = int(rows * 32);
  if (rows * cols > 4096) threads = 1024;
  threads = threads < 64 ? 64 : (threads > 1024 ? 1024 : threads);
  ech_base_kernel<<<1, threads, smem, s>>>(p, magic_of(p), int(rows), int(cols), H, ldh, W, ldw,
                                           Tc, ldt, info);
  GFQ_CUDA(cudaGetLastError());
    count_launch();
}

// ------------------------------------------------------------------ K6
namespace {
__global__ void random_fill_kernel(std::uint32_t p, std::int64_t rows,
                                   std::int64_t cols, std::uint64_t seed,
                                   std::uint64_t draw0, std::int64_t draw_ld, std::uint64_t limit,
                                   std::uint8_t* dst, std::int64_t ldd,
                                   std::uint32_t* rejects) {
  for (std::int64_t r = blockIdx.y; r < rows; r += gridDim.y) {
    for (std::int64_t c = blockIdx.x * blockDim.x + threadIdx.x; c < cols;
         c += std::int64_t(gridDim.x) * blockDim.x) {
      const std::uint64_t t = draw0 + std::uint64_t(r) * std::uint64_t(draw_ld) + std::uint64_t(c);
      std::uint64_t z = seed + (t + 1) * 0x9e3779b97f4a7c15ULL;
      z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
      z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
      z = z ^ (z >> 31);
      if (z >= limit && rejects) atomicAdd(rejects, 1u);
      dst[r * ldd + c] = p <= 1 ? 0 : std::uint8_t(z % p);
    }
  }
}
}  // namespace

void random_fill(std::uint32_t p, std::int64_t rows, std::int64_t cols,
                 std::uint64_t seed, std::uint64_t draw0, std::int64_t draw_ld,
                 std::uint8_t* dst, std::int64_t ldd, std::uint32_t* rejects, cudaStream_t s) {
  if (rows == 0 || cols == 0) return;
  const std::uint64_t limit = p <= 1 ? ~0ULL : (~0ULL - (~0ULL % p));
  const unsigned gx = unsigned((cols + 255) / 256 < 64 ? (cols + 255) / 256 : 64);
  const unsigned gy = unsigned(rows < 65535 ? rows : 65535);
  random_fill_kernel<<<dim3(gx, gy), 256, 0, s>>>(p, rows, cols, seed, draw0, draw_ld, limit, dst,
                                                   ldd, rejects);
  GFQ_CUDA(cudaGetLastError());
    count_launch();
}

}  // namespace gfq::dev
