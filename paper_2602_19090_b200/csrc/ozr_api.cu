// ozr_api.cu — the C ABI (include/ozr.h) and the host orchestration of one refinement sweep:
// parameter choice (β, digit budgets, pair plans), kernel launches on the context stream, and the
// few device->host reads of scalars the choices depend on. No math of the method runs on the host
// except the choice of β (§4.1 lines 458-463 / §3.3) from O(n) statistics.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/ozr.h"
#include "certify.h"
#include "syev.h"
#include "comm.h"
#include "kernels.h"
#include "ozr_internal.h"

using namespace ozr;

namespace {

constexpr double kU = 0x1p-53;
constexpr int kBetaMin = 2, kBetaMax = 52;
constexpr int kMaxDigits = 15;
constexpr int kMaxBands = 8;

int64_t round16(int64_t x) { return (x + 15) / 16 * 16; }

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
};
// Guard-band mode (OZR_GUARD=1 at ozr_create; memory-safety checking without compute-sanitizer): every workspace
// buffer gets kGuardBytes of a fixed pattern behind its end, checked after every ABI call that ran kernels.
constexpr size_t kGuardBytes = 4096;
constexpr unsigned char kGuardByte = 0xA5;

}  // namespace

struct ozr_ctx_s {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  std::vector<DevBuf> bufs;
  std::vector<int> last_members, last_offsets{0};  // unresolved groups of the last sweep (R13)
  cudaEvent_t ev[10];
  const double* last_R = nullptr;  // form_R: R of the last sweep (workspace), n x nl
  int64_t last_R_n = 0, last_R_nl = 0;
  cudaStream_t xstream = nullptr;  // side stream of the digit all-gather (overlaps the V product)
  cudaEvent_t ev_sync = nullptr;   // the host waits on this instead of the whole stream
  cudaEvent_t xev[2];
  // column-band pipeline of the slice products (run_banded): the recombination of band b runs on rstream
  // while the main stream computes the GEMM of band b + 1
  cudaStream_t rstream = nullptr;
  cudaEvent_t bev[kMaxBands + 2];
  SyevWorkspace syev;  // the hand-written dense eigensolver of the large-group sub-solve (syev.cu)
  // Host staging of the sweep's small reads and writes (mapped pinned memory, moved by a kernel — not by a
  // copy engine, which may be busy with a caller's large transfers on another stream): d2h() queues a read
  // that lands in `dst` at the next flush(), after the synchronisation that covers it.
  char* hst = nullptr;
  size_t hst_cap = 0, hst_off = 0;
  struct Pend {
    void* dst;
    const char* src;
    size_t n;
  };
  std::vector<Pend> pend;
  int staged_launches = 0;  // k_copy_bytes launches of the current sweep (counted in the step report)
  char* stage(size_t bytes) {
    const size_t off = (hst_off + 15) & ~static_cast<size_t>(15);
    if (off + bytes > hst_cap) return nullptr;
    hst_off = off + bytes;
    return hst + off;
  }
  bool d2h(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    char* st = stage(bytes);
    if (!st) return false;
    ozr::launch_copy_bytes(st, src, bytes, s);
    pend.push_back({dst, st, bytes});
    ++staged_launches;
    return true;
  }
  bool h2d(void* ddst, const void* src, size_t bytes, cudaStream_t s) {
    char* st = stage(bytes);
    if (!st) return false;
    memcpy(st, src, bytes);
    ozr::launch_copy_bytes(ddst, st, bytes, s);
    ++staged_launches;
    return true;
  }
  void flush() {
    for (auto& p : pend) memcpy(p.dst, p.src, p.n);
    pend.clear();
    hst_off = 0;
  }
  bool events = false;
  // tracing (OZR_TRACE=1): named events between the kernels of a sweep, printed to stderr per sweep
  bool trace = false;
  std::vector<cudaEvent_t> tev;
  std::vector<const char*> tname;
  std::vector<double> thost;  // host wall clock (ms) when the mark was recorded
  int tn = 0;
  void mark(const char* name) {
    if (!trace) return;
    if (tn >= static_cast<int>(tev.size())) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      tev.push_back(e);
      tname.push_back(name);
      thost.push_back(0.0);
    }
    tname[tn] = name;
    thost[tn] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
    cudaEventRecord(tev[tn++], stream);
  }
  void dump() {
    if (!trace || tn < 2) {
      tn = 0;
      return;
    }
    cudaEventSynchronize(tev[tn - 1]);
    // a "~" mark is recorded just before a launch: the segment ending there is GPU time not spent in the
    // sweep's kernels (host decisions, synchronisations, small copies)
    fprintf(stderr, "[ozr trace] gpu ms between marks (host ms in brackets):");
    double gap = 0.0, tot = 0.0;
    for (int i = 1; i < tn; ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, tev[i - 1], tev[i]);
      fprintf(stderr, " %s=%.3f[%.3f]", tname[i], ms, thost[i] - thost[i - 1]);
      tot += ms;
      if (tname[i][0] == '~') gap += ms;
    }
    fprintf(stderr, " | total %.3f, between kernels %.3f\n", tot, gap);
    tn = 0;
  }

  bool guard = false;
  int guard_bad = -1;  // a slot whose guard band was found overwritten (reported by guard_check)
  bool guard_ok(const DevBuf& b) {
    unsigned char h[kGuardBytes];
    if (cudaMemcpy(h, static_cast<char*>(b.p) + b.bytes, kGuardBytes, cudaMemcpyDeviceToHost) != cudaSuccess) return false;
    for (size_t i = 0; i < kGuardBytes; ++i)
      if (h[i] != kGuardByte) return false;
    return true;
  }
  // Workspace slot: grow-only device buffer.
  template <typename T>
  T* ws(int slot, size_t count) {
    if (static_cast<int>(bufs.size()) <= slot) bufs.resize(slot + 1);
    DevBuf& b = bufs[slot];
    size_t need = count * sizeof(T);
    if (need == 0) need = 16;
    if (b.bytes < need) {
      if (b.p) {
        if (guard) cudaStreamSynchronize(stream);  // the old buffer's last users are done before it is checked
        if (guard && !guard_ok(b)) guard_bad = slot;
        cudaFree(b.p);
      }
      b.p = nullptr;
      b.bytes = 0;
      if (cudaMalloc(&b.p, need + (guard ? kGuardBytes : 0)) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
      }
      b.bytes = need;
      if (guard) {
        cudaMemset(static_cast<char*>(b.p) + need, kGuardByte, kGuardBytes);
        cudaDeviceSynchronize();
      }
    }
    return static_cast<T*>(b.p);
  }
};

namespace {

enum Slot {
  S_ADIG, S_AELL, S_W, S_X1, S_XDIG, S_XDIGT, S_G, S_SH, S_SL, S_RH, S_RL, S_PLANES, S_VH, S_VL, S_LAM, S_ER,
  S_ERR, S_EMAX, S_RDIG, S_RELL, S_EP, S_NRM2, S_NU2, S_WNEXT, S_ZEROELL, S_TMP1, S_TMP2, S_BELL, S_AT, S_ONES,
  S_EDGES, S_ECOUNT, S_CINT, S_CDBL, S_CM, S_CR, S_CK, S_CV, S_CZ, S_CT, S_CSCR, S_CFLAG, S_SCAL, S_UFALL, S_CPART, S_GCNT, S_WA, S_GPLANES, S_RMAT, S_NR2, S_NW2, S_DWORK, S_DINFO, S_PI_V, S_PI_Z, S_PI_Y, S_PI_P, S_PI_S, S_CXG, S_CGJ, S_CGP,
  S_CEB, S_CCB, S_CSE, S_CSC, S_CESQ, S_CDSQ, S_CFLG, S_CEBT, S_CRE, S_OZA, S_OZB, S_OZEA, S_OZEB, S_OZT, S_OZP, S_DP, S_DTZ, S_DTH, S_PI_LZ, S_PI_U, S_PI_T,
  S_HXS, S_HX1, S_HMA, S_HVH, S_HVL, S_HR2, S_HW, S_HB, S_HQ, S_HUH, S_HUL, S_HV1, S_HV2, S_HV3, S_HV4, S_HXD, S_HG,
  S_HSH, S_HSL, S_HRH, S_HRL
};

ozr_status fail(ozr_ctx c, ozr_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  return st;
}

ozr_status cuda_check(ozr_ctx c, cudaError_t e, const char* what) {
  if (e == cudaSuccess) return OZR_OK;
  cudaGetLastError();
  return fail(c, e == cudaErrorMemoryAllocation ? OZR_ERR_NOMEM : OZR_ERR_CUDA, "%s: %s", what,
              cudaGetErrorString(e));
}

#define OZR_CK(expr, what)                                  \
  do {                                                      \
    ozr_status st__ = cuda_check(ctx, (expr), (what));      \
    if (st__ != OZR_OK) return st__;                        \
  } while (0)
// staged small transfers; a transfer larger than the staging area (the cluster branch's packed upload for
// very large groups) falls back to a plain (synchronous, pageable) copy
#define OZR_D2H(dst, src, bytes)                                                                               \
  do {                                                                                                         \
    if (!ctx->d2h((dst), (src), (bytes), s))                                                                   \
      OZR_CK(cudaMemcpyAsync((dst), (src), (bytes), cudaMemcpyDeviceToHost, s), "D2H");                     \
  } while (0)
#define OZR_H2D(dst, src, bytes)                                                                               \
  do {                                                                                                         \
    if (!ctx->h2d((dst), (src), (bytes), s))                                                                   \
      OZR_CK(cudaMemcpyAsync((dst), (src), (bytes), cudaMemcpyHostToDevice, s), "H2D");                     \
  } while (0)
#define OZR_ALLOC(ptr)                                                        \
  do {                                                                        \
    if (!(ptr)) return fail(ctx, OZR_ERR_NOMEM, "workspace allocation failed"); \
  } while (0)

// ---------------------------------------------------------------- pair / group planning (R7)
struct Group {
  int d;
  std::vector<std::pair<int, int>> pairs;  // 1-based (s, t)
};

int64_t pair_cap(int64_t K) {
  const int64_t c = (int64_t(2147483647)) / (K * 16384);
  return c < 1 ? 1 : c;
}

std::vector<Group> plan_groups(int kA, int kB, int L, int64_t K) {
  std::vector<Group> out;
  const int64_t cap = pair_cap(K);
  const int dmax = std::min(L, kA + kB);
  for (int d = 2; d <= dmax; ++d) {
    std::vector<std::pair<int, int>> pairs;
    for (int s = 1; s <= kA; ++s) {
      const int t = d - s;
      if (t >= 1 && t <= kB) pairs.push_back({s, t});
    }
    for (size_t i = 0; i < pairs.size(); i += cap) {
      Group g;
      g.d = d;
      for (size_t q = i; q < pairs.size() && q < i + cap; ++q) g.pairs.push_back(pairs[q]);
      out.push_back(g);
    }
  }
  return out;
}

int count_pairs(const std::vector<Group>& gs) {
  int n = 0;
  for (auto& g : gs) n += static_cast<int>(g.pairs.size());
  return n;
}

bool make_tables(const std::vector<Group>& gs, int L, int64_t K, PairTable& pt, RecombPlan& rp) {
  if (gs.empty() || static_cast<int>(gs.size()) > kMaxGroups || static_cast<int>(gs.size()) > kPlanGroups) return false;
  if (count_pairs(gs) > kMaxPairs) return false;
  memset(&pt, 0, sizeof pt);
  memset(&rp, 0, sizeof rp);
  int np = 0;
  for (size_t g = 0; g < gs.size(); ++g) {
    pt.first[g] = np;
    pt.out_plane[g] = static_cast<int>(g);
    pt.diag[g] = gs[g].d;
    for (auto& st : gs[g].pairs) {
      pt.s[np] = static_cast<unsigned char>(st.first - 1);
      pt.t[np] = static_cast<unsigned char>(st.second - 1);
      ++np;
    }
    rp.diag[g] = gs[g].d;
  }
  pt.first[gs.size()] = np;
  pt.ngroups = static_cast<int>(gs.size());
  rp.ngroups = pt.ngroups;
  rp.L = L;
  // chunks: T_c must fit an int128: bits(C) + log2(groups in chunk) + 1 + 8(d_last − d_first) ≤ 125
  double cbits = std::log2(static_cast<double>(K) * 16384.0 * static_cast<double>(pair_cap(K)) + 1.0);
  cbits = std::min(cbits, 31.0);
  int nc = 0;
  size_t g = 0;
  while (g < gs.size()) {
    if (nc >= kMaxChunks) return false;
    rp.chunk_first[nc] = static_cast<int>(g);
    const int d0 = gs[g].d;
    size_t h = g + 1;
    while (h < gs.size()) {
      const double bits = cbits + std::ceil(std::log2(static_cast<double>(h - g + 1))) + 1.0 + 8.0 * (gs[h].d - d0);
      if (bits > 125.0) break;
      ++h;
    }
    ++nc;
    g = h;
  }
  rp.chunk_first[nc] = static_cast<int>(gs.size());
  rp.nchunks = nc;
  // fast path: one int128 with the zero-padded limbs: 31 + 8·(4·⌈G/4⌉ − 1) + 2 ≤ 121 bits for G ≤ 12
  rp.consecutive = (gs.size() <= 12 && nc == 1) ? 1 : 0;
  for (size_t q = 0; q < gs.size(); ++q)
    if (gs[q].d != gs[0].d + static_cast<int>(q)) rp.consecutive = 0;
  return true;
}

// Smallest L such that dropping diagonals d > L costs ≤ tau (statistical √K bound, R8):
// diagonal d contributes ≤ np(d) · 2√K · 2^14 · 2^{eA + eB + 4 − 8d} to every |c_ij|.
int choose_L(int kA, int kB, int64_t K, int eA, int eB, double tau) {
  for (int L = 2; L < kA + kB; ++L) {
    double tail = 0.0;
    for (int d = L + 1; d <= kA + kB; ++d) {
      int np = 0;
      for (int s = 1; s <= kA; ++s)
        if (d - s >= 1 && d - s <= kB) ++np;
      tail += np * 2.0 * std::sqrt(static_cast<double>(K)) * std::ldexp(1.0, 14 + eA + eB + 4 - 8 * d);
    }
    if (tail <= tau) return L;
  }
  return kA + kB;
}

// Everything the planner needs from one λ̂ vector, from ONE ordering (ascending λ̂, ties by index; no sort
// at all when λ̂ is already ascending, the usual case): gap0 = min neighbour fl-difference,
// gap_pos = the smallest positive one (R16), colgap_j = min_{i≠j} |λ̂_i − λ̂_j| (R8b), max|λ̂|.
struct LamStats {
  double gap0 = INFINITY, gap_pos = 0.0, maxabs = 0.0;
  std::vector<double> colgap;
};

LamStats lam_stats(const std::vector<double>& lam) {
  const size_t n = lam.size();
  LamStats st;
  std::vector<int> idx(n);
  for (size_t i = 0; i < n; ++i) idx[i] = static_cast<int>(i);
  bool sorted = true;
  for (size_t i = 1; i < n && sorted; ++i) sorted = !(lam[i] < lam[i - 1]);
  if (!sorted)
    std::sort(idx.begin(), idx.end(), [&](int a, int b) { return lam[a] < lam[b] || (lam[a] == lam[b] && a < b); });
  st.colgap.assign(n, INFINITY);
  double gp = INFINITY;
  for (size_t p = 0; p < n; ++p) {
    st.maxabs = std::max(st.maxabs, std::fabs(lam[p]));
    if (p > 0) {
      const double d = lam[idx[p]] - lam[idx[p - 1]];
      st.gap0 = std::min(st.gap0, d);
      if (d > 0.0) gp = std::min(gp, d);
      st.colgap[idx[p]] = std::min(st.colgap[idx[p]], d);
      st.colgap[idx[p - 1]] = std::min(st.colgap[idx[p - 1]], d);
    }
  }
  st.gap_pos = std::isfinite(gp) ? gp : std::max(st.maxabs * kU, 1e-300);
  return st;
}


// The first pair of exactly equal estimates in ascending (λ̂, index) order (for the error message when the
// cluster branch is off; PAPER.md:333 assumes distinct eigenvalues). Returns false when all are distinct.
bool equal_pair(const std::vector<double>& lam, int* a, int* b) {
  std::vector<int> idx(lam.size());
  for (size_t i = 0; i < lam.size(); ++i) idx[i] = static_cast<int>(i);
  std::sort(idx.begin(), idx.end(), [&](int x, int y) { return lam[x] < lam[y] || (lam[x] == lam[y] && x < y); });
  for (size_t q = 1; q < idx.size(); ++q)
    if (lam[idx[q]] == lam[idx[q - 1]]) {
      *a = idx[q - 1];
      *b = idx[q];
      return true;
    }
  return false;
}

int pairs_upto(int kA, int kB, int L) {
  int np = 0;
  for (int s = 1; s <= kA; ++s)
    for (int t = 1; t <= kB; ++t)
      if (s + t <= L) ++np;
  return np;
}

// R8b: per-N-tile pair budgets. Column j of V = A·X̂ and of W = X̂ᵀRes only has to be accurate to
// θ·δ'·gap_j (an error η in w_ij moves ẽ_ij by η/|λ_j − λ_i| ≤ η/gap_j), so each 256-column tile gets
// the smallest L that meets the tightest column of the tile. Returns the max L over tiles and fills
// tileL; *int8_pairs receives Σ_tiles pairs(L_t)·(tile width) / n (the average pairs per column).
int tile_budgets(int kA, int kB, int64_t K, int eA, const std::vector<int>& eB_col, const std::vector<double>& tau_col,
                 unsigned char* tileL, double* avg_pairs) {
  const int64_t n = static_cast<int64_t>(tau_col.size());
  const int64_t nt = (n + kTileN - 1) / kTileN;
  int Lmax = 2;
  double pw = 0.0;
  // choose_L's tail sums with eA + eB factored out: every term carries the same power of two, so
  // ldexp(base[L], eA + eB) is bit-for-bit the sum choose_L forms (exact scaling), once per product instead of
  // once per tile
  std::vector<double> base(kA + kB + 1, 0.0);
  for (int L = 2; L < kA + kB; ++L) {
    double tail = 0.0;
    for (int d = L + 1; d <= kA + kB; ++d) {
      int np = 0;
      for (int s = 1; s <= kA; ++s)
        if (d - s >= 1 && d - s <= kB) ++np;
      tail += np * 2.0 * std::sqrt(static_cast<double>(K)) * std::ldexp(1.0, 14 + 4 - 8 * d);
    }
    base[L] = tail;
  }
  std::vector<int> pairs_of(kA + kB + 1, 0);
  for (int L = 2; L <= kA + kB; ++L) pairs_of[L] = pairs_upto(kA, kB, L);
  auto choose = [&](int eB, double tau) {
    for (int L = 2; L < kA + kB; ++L)
      if (std::ldexp(base[L], eA + eB) <= tau) return L;
    return kA + kB;
  };
  for (int64_t t = 0; t < nt; ++t) {
    double tau = INFINITY;
    int eB = -100000;
    const int64_t j1 = std::min<int64_t>(n, (t + 1) * kTileN);
    for (int64_t j = t * kTileN; j < j1; ++j) {
      tau = std::min(tau, tau_col[j]);
      eB = std::max(eB, eB_col[j]);
    }
    int L = (eB == -100000) ? 2 : choose(eB, tau);
    L = std::max(2, std::min(L, kA + kB));
    tileL[t] = static_cast<unsigned char>(L);
    Lmax = std::max(Lmax, L);
    pw += static_cast<double>(pairs_of[L]) * static_cast<double>(j1 - t * kTileN);
  }
  *avg_pairs = pw / static_cast<double>(n);
  return Lmax;
}

// Average number of int32 group planes the recombination of one element reads (the per-tile budgets skip the
// groups above a tile's L): the algorithmic plane bytes of a recombination kernel are 4 × this per element.
double avg_planes(const RecombPlan& rp, int64_t n) {
  if (!rp.tile_budgets) return rp.ngroups;
  double acc = 0.0;
  for (int64_t t = 0; t * kTileN < n; ++t) {
    int c = 0;
    for (int g = 0; g < rp.ngroups; ++g) c += rp.diag[g] <= rp.tileL[t];
    acc += static_cast<double>(c) * static_cast<double>(std::min<int64_t>(kTileN, n - t * kTileN));
  }
  return acc / static_cast<double>(n);
}

void apply_tiles(PairTable& pt, RecombPlan& rp, const unsigned char* tileL, int64_t n) {
  const int64_t nt = (n + kTileN - 1) / kTileN;
  pt.tile_budgets = 1;
  rp.tile_budgets = 1;
  for (int64_t t = 0; t < nt; ++t) pt.tileL[t] = rp.tileL[t] = tileL[t];
}

// Digits needed so that the fixed-point LSB 2^{e − S_k} ≤ 2^{lsb_max} (k clamped to [1, 15]).
int digits_for(int emax, int lsb_max) {
  int k = 1;
  while (k < kMaxDigits && (emax - (8 * (k - 1) + 6)) > lsb_max) ++k;
  return k;
}

int kx_for_beta(int beta) {
  int k = 1;
  while (8 * (k - 1) + 6 < 53 - beta) ++k;
  return k;
}

int ceil_log2_host(double v) {
  if (v == 0.0) return 0;
  int e;
  const double m = std::frexp(v, &e);
  return (m == 0.5) ? e - 1 : e;
}

// β of §4.1 (mode 0) / §3.3 (mode 1) / §4.3 sparse (mode 2: γ·min(k, √n) in place of
// √(nδ·gap/max|λ̂|), i.e. the §4.1 form with n → min(k², n)), evaluated in the operation order of R3.
int choose_beta(int64_t n, double delta_p, int mode, double xi, double gap, double maxlam, double ssum,
                int64_t row_nnz) {
  const int64_t k = (row_nnz > 0 && row_nnz < n) ? row_nnz : n;
  const double c = (mode == 0) ? static_cast<double>(n)
                   : (mode == 2) ? static_cast<double>(std::min<int64_t>(k * k, n))
                                 : (xi > 0 ? xi : static_cast<double>(n));
  const double t = ((c * delta_p) * gap) / (maxlam * ssum);
  const double Z = std::sqrt(t) / (0.75 * kU);
  int e;
  const double m = std::frexp(Z, &e);
  if (mode != 1) return e - 1;         // ⌊log2 Z⌋
  return (m == 0.5) ? e - 1 : e;       // ⌈log2 Z⌉
}

int alpha_dense(int64_t n, int beta) {
  int c = 0;
  while ((int64_t(1) << (2 * c)) < n) ++c;
  return 53 - beta + c;
}



// ---------------------------------------------------------------- cluster branch (R13): host grouping
// Connected components of the unresolved-pair graph; members sorted by (λ̂, index), groups by first member.
// root[i]: the (flattened) device union-find label of column i.
void unresolved_groups(int64_t n, const std::vector<int>& root, const std::vector<double>& lam,
                       std::vector<int>& members, std::vector<int>& offsets) {
  std::vector<int> cnt(n, 0);
  for (int64_t i = 0; i < n; ++i) ++cnt[root[i]];
  std::vector<int> slot(n, -1);
  std::vector<std::vector<int>> comp;
  for (int64_t i = 0; i < n; ++i)
    if (cnt[root[i]] >= 2) {
      if (slot[root[i]] < 0) {
        slot[root[i]] = static_cast<int>(comp.size());
        comp.emplace_back();
      }
      comp[slot[root[i]]].push_back(static_cast<int>(i));
    }
  std::vector<std::vector<int>> groups;
  for (auto& cg : comp) {
    std::vector<int> g = cg;
    std::sort(g.begin(), g.end(), [&](int a, int b) { return lam[a] < lam[b] || (lam[a] == lam[b] && a < b); });
    groups.push_back(g);
  }
  std::sort(groups.begin(), groups.end(), [](const std::vector<int>& a, const std::vector<int>& b) { return a[0] < b[0]; });
  members.clear();
  offsets.assign(1, 0);
  for (auto& g : groups) {
    members.insert(members.end(), g.begin(), g.end());
    offsets.push_back(static_cast<int>(members.size()));
  }
}

// Σ_j 2^{2⌈log2 w_j⌉} added in ascending exponent order (R3), via a histogram of the exponents.
double sum_pow2_2c(const std::vector<double>& w) {
  std::vector<int> cnt(2200, 0);
  for (double x : w)
    if (x != 0.0) ++cnt[ceil_log2_host(x) + 1100];
  double s = 0.0;
  for (int c = 0; c < 2200; ++c)
    for (int q = 0; q < cnt[c]; ++q) s = s + std::ldexp(1.0, 2 * (c - 1100));
  return s;
}

// Slice GEMM `idx` (0: V, 1: W, 2: U, 3: G = X̂ᵀX̂ with form_R) of a sweep, bracketed by events ev[2+2idx], ev[3+2idx]
// (read after the sweep's final synchronisation; no extra host sync here).
ozr_status run_gemm(ozr_ctx ctx, const DigitOperand& A, const DigitOperand& B, int M, int N, int K,
                    const PairTable& pt, int32_t* planes, int idx) {
  cudaEventRecord(ctx->ev[2 + 2 * idx], ctx->stream);
  int* cnt = ctx->ws<int>(S_GCNT, 4);
  OZR_ALLOC(cnt);
  OZR_CK(launch_gemm_i8(A, B, M, N, K, pt, planes, static_cast<int64_t>(M) * N, M, ctx->stream, cnt), "slice GEMM");
  cudaEventRecord(ctx->ev[3 + 2 * idx], ctx->stream);
  return OZR_OK;
}

// Column bands of a slice product and its recombination: band b of the output (columns
// [c0, c1), multiples of the 256-column tile) only needs band b of the right operand, so the GEMM of band
// b + 1 (main stream) runs while the recombination of band b runs on ctx->rstream. The GEMM holds 197 KB of
// shared memory on every SM, so the overlapped recombinations take the register path (a few KB); the
// last band, which nothing overlaps, takes the TMA-staged path. Same arithmetic per column either way.
// Measured on B200 (c4', n = 8192): OFF by default. The register-path recombination CTAs do co-reside with
// the persistent GEMM (a trivial kernel on the side stream completes at once) but starve behind the GEMM's
// TMA traffic: band b's recombine_V takes 4.5 ms instead of 0.5, the band GEMMs lose ~5 %, and the sweep
// goes from 28.4 to 29.4 ms. OZR_BANDS=k (k ≤ 8) enables k bands for experiments.
int band_count(int64_t nl) {
  const char* v = getenv("OZR_BANDS");
  const int want = v ? atoi(v) : 1;
  int nb = static_cast<int>(std::min<int64_t>(want, nl / 1024));
  return std::max(1, std::min(nb, kMaxBands));
}

ozr_status run_banded(ozr_ctx ctx, const DigitOperand& A, const DigitOperand& B, int M, int N, int K,
                      const PairTable& pt, int32_t* planes, int idx,
                      const std::function<void(int64_t c0, int64_t c1, int tile0, int tma, cudaStream_t st)>& recomb,
                      const std::function<void(cudaStream_t st)>& side_first = nullptr) {
  cudaStream_t s = ctx->stream, r = ctx->rstream;
  const int nb = band_count(N);
  const int64_t tiles = (N + kTileN - 1) / kTileN;
  const int64_t tpb = (tiles + nb - 1) / nb;  // tiles per band
  int* cnt = ctx->ws<int>(S_GCNT, 4);
  OZR_ALLOC(cnt);
  cudaEventRecord(ctx->ev[2 + 2 * idx], s);
  OZR_CK(cudaEventRecord(ctx->bev[kMaxBands], s), "event");
  OZR_CK(cudaStreamWaitEvent(r, ctx->bev[kMaxBands], 0), "wait");  // the side stream sees all earlier work
  if (side_first) side_first(r);  // independent work that overlaps the first band's GEMM
  int b = 0;
  for (int64_t t0 = 0; t0 < tiles; t0 += tpb, ++b) {
    const int64_t c0 = t0 * kTileN, c1 = std::min<int64_t>(N, (t0 + tpb) * kTileN);
    PairTable ptb = pt;
    if (pt.tile_budgets)
      for (int64_t t = t0; t < std::min<int64_t>(tiles, t0 + tpb); ++t) ptb.tileL[t - t0] = pt.tileL[t];
    DigitOperand Bb{B.base + c0 * B.ld, B.ld, B.plane_stride, B.nplanes};
    OZR_CK(launch_gemm_i8(A, Bb, M, static_cast<int>(c1 - c0), K, ptb, planes + c0 * M,
                          static_cast<int64_t>(M) * N, M, s, cnt, A.nplanes > B.nplanes ? 3 : 1),
           "slice GEMM band");
    const bool last = c1 >= N;
    if (last) {
      cudaEventRecord(ctx->ev[3 + 2 * idx], s);
      recomb(c0, c1, static_cast<int>(t0), 1, s);
    } else {
      OZR_CK(cudaEventRecord(ctx->bev[b], s), "event");
      OZR_CK(cudaStreamWaitEvent(r, ctx->bev[b], 0), "wait");
      recomb(c0, c1, static_cast<int>(t0), 0, r);
    }
  }
  OZR_CK(cudaGetLastError(), "recombination band");
  OZR_CK(cudaEventRecord(ctx->bev[kMaxBands + 1], r), "event");
  OZR_CK(cudaStreamWaitEvent(s, ctx->bev[kMaxBands + 1], 0), "join");
  return OZR_OK;
}

// a RecombPlan whose per-tile budgets start at tile t0 (the band's first tile)
RecombPlan shift_plan(const RecombPlan& rp, int t0) {
  RecombPlan q = rp;
  if (rp.tile_budgets)
    for (int t = 0; t + t0 < 256; ++t) q.tileL[t] = rp.tileL[t + t0];
  return q;
}

ozr_status err_bits(ozr_ctx ctx, int h) {
  if (h & ERR_SOLVER) return fail(ctx, OZR_ERR_CUDA, "dense cluster sub-solve: the eigensolver reported failure");
  if (h & ERR_NONFINITE) return fail(ctx, OZR_ERR_NONFINITE, "non-finite value in an input matrix");
  if (h & ERR_RANGE) return fail(ctx, OZR_ERR_RANGE, "exponent range exceeded in the digit split");
  if (h & ERR_DEGENERATE)
    return fail(ctx, OZR_ERR_DEGENERATE, "degenerate column or equal eigenvalue estimates (PAPER.md:333)");
  return OZR_OK;
}

ozr_status read_err(ozr_ctx ctx, int* derr) {
  int h = 0;
  OZR_CK(cudaMemcpyAsync(&h, derr, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream), "D2H err");
  OZR_CK(cudaStreamSynchronize(ctx->stream), "sync");
  if (h & ERR_NONFINITE) return fail(ctx, OZR_ERR_NONFINITE, "non-finite value in an input matrix");
  if (h & ERR_RANGE) return fail(ctx, OZR_ERR_RANGE, "exponent range exceeded in the digit split");
  if (h & ERR_DEGENERATE)
    return fail(ctx, OZR_ERR_DEGENERATE, "degenerate column or equal eigenvalue estimates (PAPER.md:333)");
  return OZR_OK;
}

// ---------------------------------------------------------------- one sweep (internal)
struct SweepState {
  // A split (reused across sweeps of one ozr_refine_to_tol call)
  const double* A = nullptr;
  int64_t nA = 0;
  int kA_split = 0;
  int eA_max = 0;
  bool have_w = false;  // wnext valid (column maxima of the current X)
};

// A → digit planes (a1), stream-ordered; the exponents land in `hell` (host) at the caller's next
// synchronisation, after which split_A_finish derives e_A,max. Error flags go to derr.
ozr_status split_A_launch(ozr_ctx ctx, const double* A, int64_t n, int64_t lda, int kA, int* derr,
                          std::vector<int32_t>& /*hell*/) {
  const int64_t ld = round16(n);
  int8_t* adig = ctx->ws<int8_t>(S_ADIG, static_cast<size_t>(kA) * ld * n);
  int32_t* aell = ctx->ws<int32_t>(S_AELL, n);
  OZR_ALLOC(adig);
  OZR_ALLOC(aell);
  // A symmetric: its columns are its rows, so the COLWISE split of A is the row-wise split of the
  // A operand of V = A·X̂ (K-major) and ℓ_i is its per-row exponent.
  launch_split_fixed(A, nullptr, lda, static_cast<int>(n), static_cast<int>(n), kA, adig, ld, ld * n, aell, derr,
                     ctx->stream);
  OZR_CK(cudaGetLastError(), "split A");
  return OZR_OK;
}

// e_A,max = max_i ℓ_i + S_kA = max_i ⌈log2 max_j |a_ij|⌉ (the split's per-line exponent, 0 for a zero line)
void split_A_finish(const double* A, int64_t n, const std::vector<double>& hwA, int kA, SweepState& st) {
  int em = -100000;
  for (int64_t i = 0; i < n; ++i) em = std::max(em, hwA[i] != 0.0 ? ceil_log2_host(hwA[i]) : 0);
  st.A = A;
  st.nA = n;
  st.kA_split = kA;
  st.eA_max = em;
}

// FP64-accurate product C = A·B (m x k times k x n, column-major, fp64 result) on the INT8 slice GEMM for the
// dense sub-solve of large unresolved groups (R13): A split per row, B per column into kOzDig digits, digit pairs
// s + t ≤ kOzDig + 1 (dropped pairs below 2^{-8·kOzDig+...} of max|A_i,:|·max|B_:,j|·k), exact recombination
// rounded once. a_trans: A is stored as its transpose (k x m, lda) — e.g. a symmetric matrix — so the per-row
// split of A is the per-column split of the stored matrix (no transpose).
// Own workspace slots (the sweep's digit buffers stay live); split error flags accumulate into derr.
constexpr int kOzDig = 8;
constexpr int kSyevBigGemm = 1024;  // dense eigensolver products with a dimension ≥ this run on the INT8 slice GEMM
ozr_status oz_dgemm(ozr_ctx ctx, int64_t m, int64_t n, int64_t k, const double* A, int64_t lda, bool a_trans,
                    const double* B, int64_t ldb, double* C, int64_t ldc, int* derr) {
  cudaStream_t s = ctx->stream;
  const int64_t ldk = round16(k);
  const int kd = kOzDig, L = kOzDig + 1;
  int8_t* da = ctx->ws<int8_t>(S_OZA, static_cast<size_t>(kd) * ldk * m);
  int8_t* db = ctx->ws<int8_t>(S_OZB, static_cast<size_t>(kd) * ldk * n);
  int32_t* ea = ctx->ws<int32_t>(S_OZEA, m);
  int32_t* eb = ctx->ws<int32_t>(S_OZEB, n);
  OZR_ALLOC(da); OZR_ALLOC(db); OZR_ALLOC(ea); OZR_ALLOC(eb);
  const double* As = A;
  int64_t lds = lda;
  if (!a_trans) {  // rows of A as columns: Aᵀ (k x m)
    double* T = ctx->ws<double>(S_OZT, static_cast<size_t>(k) * m);
    OZR_ALLOC(T);
    launch_transpose_f64(A, lda, T, k, static_cast<int>(m), static_cast<int>(k), s);
    As = T;
    lds = k;
  }
  launch_split_fixed(As, nullptr, lds, static_cast<int>(k), static_cast<int>(m), kd, da, ldk, ldk * m, ea, derr, s);
  launch_split_fixed(B, nullptr, ldb, static_cast<int>(k), static_cast<int>(n), kd, db, ldk, ldk * n, eb, derr, s);
  std::vector<Group> gs = plan_groups(kd, kd, L, k);
  PairTable pt;
  RecombPlan rp;
  if (!make_tables(gs, L, k, pt, rp)) return fail(ctx, OZR_ERR_RANGE, "dense sub-solve product plan too large");
  const size_t mn = static_cast<size_t>(m) * n;
  int32_t* planes = ctx->ws<int32_t>(S_OZP, static_cast<size_t>(pt.ngroups) * mn);
  int* cnt = ctx->ws<int>(S_GCNT, 4);
  OZR_ALLOC(planes); OZR_ALLOC(cnt);
  const DigitOperand oa{da, ldk, ldk * m, kd}, ob{db, ldk, ldk * n, kd};
  OZR_CK(launch_gemm_i8(oa, ob, static_cast<int>(m), static_cast<int>(n), static_cast<int>(k), pt, planes,
                        static_cast<int64_t>(mn), m, s, cnt),
         "dense sub-solve slice GEMM");
  launch_recombine_dd(planes, static_cast<long long>(mn), static_cast<int>(m), static_cast<int>(n), rp, ea, eb,
                      8 * (2 * kd - L), C, nullptr, ldc, s);
  OZR_CK(cudaGetLastError(), "dense sub-solve recombination");
  return OZR_OK;
}

// The Hermitian sweep's products (ozr_refine_step_herm, R18): C = A·B with explicit digit budgets (A per row into
// kA digits, B per column into kB, pairs s + t ≤ L), exact recombination rounded once to double-double (Cl
// nullable). a_trans: A stored as its transpose (k x m). Uses the dense sub-solve's product slots (the Hermitian
// step has no cluster branch). *pairs += the pair count.
ozr_status herm_product(ozr_ctx ctx, int64_t m, int64_t n, int64_t k, const double* A, int64_t lda, bool a_trans,
                        const double* B, int64_t ldb, int kA, int kB, int L, double* Ch, double* Cl, int64_t ldc,
                        int* derr, int* pairs) {
  cudaStream_t s = ctx->stream;
  const int64_t ldk = round16(k);
  int8_t* da = ctx->ws<int8_t>(S_OZA, static_cast<size_t>(kA) * ldk * m);
  int8_t* db = ctx->ws<int8_t>(S_OZB, static_cast<size_t>(kB) * ldk * n);
  int32_t* ea = ctx->ws<int32_t>(S_OZEA, m);
  int32_t* eb = ctx->ws<int32_t>(S_OZEB, n);
  OZR_ALLOC(da); OZR_ALLOC(db); OZR_ALLOC(ea); OZR_ALLOC(eb);
  const double* As = A;
  int64_t lds = lda;
  if (!a_trans) {
    double* T = ctx->ws<double>(S_OZT, static_cast<size_t>(k) * m);
    OZR_ALLOC(T);
    launch_transpose_f64(A, lda, T, k, static_cast<int>(m), static_cast<int>(k), s);
    As = T;
    lds = k;
  }
  launch_split_fixed(As, nullptr, lds, static_cast<int>(k), static_cast<int>(m), kA, da, ldk, ldk * m, ea, derr, s);
  launch_split_fixed(B, nullptr, ldb, static_cast<int>(k), static_cast<int>(n), kB, db, ldk, ldk * n, eb, derr, s);
  std::vector<Group> gs = plan_groups(kA, kB, L, k);
  PairTable pt;
  RecombPlan rp;
  if (!make_tables(gs, L, k, pt, rp)) return fail(ctx, OZR_ERR_RANGE, "Hermitian product plan too large");
  *pairs += count_pairs(gs);
  const size_t mn = static_cast<size_t>(m) * n;
  int32_t* planes = ctx->ws<int32_t>(S_OZP, static_cast<size_t>(pt.ngroups) * mn);
  int* cnt = ctx->ws<int>(S_GCNT, 4);
  OZR_ALLOC(planes); OZR_ALLOC(cnt);
  const DigitOperand oa{da, ldk, ldk * m, kA}, ob{db, ldk, ldk * n, kB};
  OZR_CK(launch_gemm_i8(oa, ob, static_cast<int>(m), static_cast<int>(n), static_cast<int>(k), pt, planes,
                        static_cast<int64_t>(mn), m, s, cnt),
         "Hermitian slice GEMM");
  launch_recombine_dd(planes, static_cast<long long>(mn), static_cast<int>(m), static_cast<int>(n), rp, ea, eb,
                      8 * (kA + kB - L), Ch, Cl, ldc, s);
  OZR_CK(cudaGetLastError(), "Hermitian recombination");
  return OZR_OK;
}

// Block-column partition: rank r of P owns columns [col0, col0 + nl), nl = n/P, col0 = r·nl.
// Every column of V, Res, W, Ẽ and X̂_new depends only on its own column of X̂^(1) plus the full X̂^(1)
// (left operand of W and U) and the full λ̂, so a rank computes its columns with the slice GEMMs on
// M = n, N = nl; the exchange per sweep is: the X̂^(1) digit planes and g (all-gather), the column
// maxima w, λ̂ and a few per-rank scalars (all-gather), and — only when unresolved groups straddle
// ranks — their W_JJ / Ẽ_{:,J} blocks (all-reduce of zero-padded buffers, exact). Every host decision is
// taken from all-gathered data in the 1-GPU order, so a P-rank sweep equals the 1-GPU sweep bit for bit
// when nl is a multiple of the 256-column tile.
ozr_status sweep(ozr_ctx ctx, Exchange* ex, const double* A, int64_t n, int64_t lda, double* Xfull, int64_t ldx,
                 double* lambda, const ozr_params& P, ozr_step_report& rep, SweepState& st) {
  memset(&rep, 0, sizeof rep);
  cudaStream_t s = ctx->stream;
  const int NP = ex ? ex->P : 1, RK = ex ? ex->rank : 0;
  const int64_t nl = n / NP, col0 = RK * nl;
  const int N = static_cast<int>(n), NL = static_cast<int>(nl);
  double* X = Xfull + col0 * ldx;  // this rank's column block
  const int64_t ld = round16(n);
  const int64_t nnl = n * nl;
  cudaEventRecord(ctx->ev[0], s);
  ctx->mark("start");
  float gemm_ms = 0.f;
  double ops = 0.0;
  int nexch = 0;

  {  // host staging: the largest phase reads ~5 n-vectors (+ the P·n union-find labels)
    const size_t need = 48 * static_cast<size_t>(n) + 8 * static_cast<size_t>(NP) * n + (1 << 20);
    if (ctx->hst_cap < need) {
      OZR_CK(cudaStreamSynchronize(s), "sync");
      if (ctx->hst) cudaFreeHost(ctx->hst);
      ctx->hst = nullptr;
      ctx->hst_cap = 0;
      OZR_CK(cudaHostAlloc(reinterpret_cast<void**>(&ctx->hst), need, cudaHostAllocMapped), "host staging");
      ctx->hst_cap = need;
    }
    ctx->pend.clear();
    ctx->hst_off = 0;
    ctx->staged_launches = 0;
  }
  int* derr = ctx->ws<int>(S_ERR, 4);
  int* demax = ctx->ws<int>(S_EMAX, 4);
  int* scal = ctx->ws<int>(S_SCAL, 4 * static_cast<size_t>(NP) + 4);
  double* w = ctx->ws<double>(S_W, n);
  double* wnext = ctx->ws<double>(S_WNEXT, n);
  OZR_ALLOC(derr); OZR_ALLOC(demax); OZR_ALLOC(scal); OZR_ALLOC(w); OZR_ALLOC(wnext);
  OZR_CK(cudaMemsetAsync(derr, 0, sizeof(int), s), "memset");

  // exchange helpers (no-ops on one GPU)
  auto xgather_on = [&](void* base, size_t bytes, cudaStream_t st_) -> ozr_status {
    if (!ex) return OZR_OK;
    ++nexch;
    if (!ex->allgather(base, bytes, st_)) return fail(ctx, OZR_ERR_COMM, "all-gather: %s", ex->err.c_str());
    return OZR_OK;
  };
  auto xgather = [&](void* base, size_t bytes) -> ozr_status { return xgather_on(base, bytes, s); };
  auto xsum = [&](double* buf, size_t count) -> ozr_status {
    if (!ex) return OZR_OK;
    ++nexch;
    if (!ex->allreduce_sum(buf, count, s)) return fail(ctx, OZR_ERR_COMM, "all-reduce: %s", ex->err.c_str());
    return OZR_OK;
  };
  // Up to 3 device ints combined over the ranks (max) plus the error flags (OR), with ONE host
  // synchronisation; pending host copies queued on the stream complete with it. Fails on error flags.
  // post (nullable): work to enqueue after the reads and before waiting for them, so that the GPU keeps
  // running it while the host takes its decisions
  auto scalars = [&](std::initializer_list<const int*> dvs, int* outs,
                     const std::function<ozr_status()>& post = nullptr) -> ozr_status {
    int k = 0;
    for (const int* dv : dvs) {
      OZR_CK(cudaMemcpyAsync(scal + 4 * RK + k, dv, sizeof(int), cudaMemcpyDeviceToDevice, s), "D2D");
      ++k;
    }
    OZR_CK(cudaMemcpyAsync(scal + 4 * RK + 3, derr, sizeof(int), cudaMemcpyDeviceToDevice, s), "D2D");
    ozr_status e = xgather(scal + 0, 4 * sizeof(int));
    if (e != OZR_OK) return e;
    std::vector<int> h(4 * NP);
    OZR_D2H(h.data(), scal, h.size() * sizeof(int));
    OZR_CK(cudaEventRecord(ctx->ev_sync, s), "event");
    if (post) {
      ozr_status pe = post();
      if (pe != OZR_OK) return pe;
    }
    OZR_CK(cudaEventSynchronize(ctx->ev_sync), "sync");
    ctx->flush();
    int bits = 0;
    for (int r = 0; r < NP; ++r) bits |= h[4 * r + 3];
    for (int q = 0; q < k; ++q) {
      outs[q] = h[q];
      for (int r = 1; r < NP; ++r) outs[q] = std::max(outs[q], h[4 * r + q]);
    }
    return err_bits(ctx, bits);
  };
#define OZR_X(expr)                     \
  do {                                  \
    ozr_status e__ = (expr);            \
    if (e__ != OZR_OK) return e__;      \
  } while (0)

  // ---- a0: statistics and parameters
  const bool fresh_w = !st.have_w;
  if (!st.have_w) {
    launch_colmax(X, ldx, N, NL, w + col0, derr, s);
    OZR_CK(cudaGetLastError(), "colmax");
  } else {
    OZR_CK(cudaMemcpyAsync(w + col0, wnext + col0, nl * sizeof(double), cudaMemcpyDeviceToDevice, s), "copy w");
  }
  OZR_X(xgather(w, nl * sizeof(double)));
  // a1 (once per call): the column maxima of A give e_A,max now; the A split itself is enqueued after the
  // a0 reads and runs while the host chooses β and the budgets
  const bool new_A = (st.A != A || st.nA != n);
  std::vector<int32_t> hell;
  std::vector<double> hwA;
  if (new_A) {
    double* wA = ctx->ws<double>(S_WA, n);
    OZR_ALLOC(wA);
    launch_colmax(A, lda, N, N, wA, derr, s);
    OZR_CK(cudaGetLastError(), "colmax A");
    hwA.resize(n);
    OZR_D2H(hwA.data(), wA, n * sizeof(double));
  }
  std::vector<double> hw(n), hlam(n);
  OZR_D2H(hw.data(), w, n * sizeof(double));
  OZR_D2H(hlam.data(), lambda, n * sizeof(double));
  OZR_X(scalars({}, nullptr, [&]() -> ozr_status {
    ctx->mark("~");
    return new_A ? split_A_launch(ctx, A, n, lda, P.kA_split, derr, hell) : OZR_OK;
  }));
  for (double x : hlam)
    if (!std::isfinite(x)) return fail(ctx, OZR_ERR_NONFINITE, "non-finite lambda");
  const double delta_p = P.delta / (P.theta > 0 ? P.theta : 1.0);
  LamStats ls_prev = lam_stats(hlam);
  const double gap0 = ls_prev.gap0;
  const double gap = (P.cluster_mode && !(gap0 > 0.0)) ? ls_prev.gap_pos : gap0;
  const double maxlam = ls_prev.maxabs;
  if (!(gap0 > 0.0) && P.cluster_mode == 0) {
    int pa = -1, pb = -1;
    equal_pair(hlam, &pa, &pb);
    return fail(ctx, OZR_ERR_DEGENERATE, "equal eigenvalue estimates λ̂_%d = λ̂_%d (gap = 0) with the cluster branch off",
                pa, pb);
  }
  const double ssum = sum_pow2_2c(hw);
  if (ssum == 0.0 || maxlam == 0.0) return fail(ctx, OZR_ERR_DEGENERATE, "zero X or zero spectrum");
  int beta_raw = (P.beta_override > 0) ? P.beta_override
                                       : choose_beta(n, delta_p, P.beta_mode, P.xi, gap, maxlam, ssum, P.row_nnz);
  int beta = std::min(std::max(beta_raw, kBetaMin), kBetaMax);
  if (!P.truncate) beta = kBetaMin;
  const int kx = kx_for_beta(beta);
  // R8: an X̂^(1) operand enters the dropped-pair tail bound with exponent c + slack, slack = S_kx − (53 − β)
  // (0..7: its leading digit is not normalised like the fixed-point splits' digits)
  const int xslack = (8 * (kx - 1) + 6) - (53 - beta);
  int cmax = -100000;
  for (double x : hw)
    if (x != 0.0) cmax = std::max(cmax, ceil_log2_host(x));
  rep.beta = beta;
  rep.beta_raw = beta_raw;
  // α (reported only): §4.1 53 − β + ⌈log2 √n⌉; §3.3 53 − β + ⌈log2 n⌉ (eq. proposed_beta); §4.3 53 − β + ⌈log2 k⌉
  rep.alpha = (P.beta_mode == 2)   ? 53 - beta + ceil_log2_host(static_cast<double>(P.row_nnz > 0 && P.row_nnz < n ? P.row_nnz : n))
              : (P.beta_mode == 1) ? 53 - beta + ceil_log2_host(static_cast<double>(n))
                                   : alpha_dense(n, beta);
  rep.kX = kx;
  rep.gap_min = gap0;
  rep.max_abs_lambda = maxlam;

  // ---- A split (once per refine_to_tol call; A and its digits are replicated on every rank)
  if (new_A) split_A_finish(A, n, hwA, P.kA_split, st);
  ctx->mark("splitA");
  // per-column accuracy of V (R8, R8b): θ_V·δ'·gap_j with the previous λ̂ (this rank's columns)
  std::vector<double>& gaps_prev = ls_prev.colgap;
  for (double& x : gaps_prev)
    if (!(x > 0.0)) x = gap;  // equal λ̂ (cluster branch): the smallest positive gap sets the budget
  std::vector<double> tau_col(nl);
  std::vector<int> c_col(nl);
  for (int64_t j = 0; j < nl; ++j) {
    tau_col[j] = P.theta_V * delta_p * (P.tile_budgets ? gaps_prev[col0 + j] : gap);
    // the X̂^(1) digits of column j sit on the grid 2^{g_j}, g_j = c_j + β − 53, with S_kx ≥ 53 − β bits:
    // for the tail bound of choose_L their "line exponent" is g_j + S_kx = c_j + slack (R8)
    c_col[j] = hw[col0 + j] != 0.0 ? ceil_log2_host(hw[col0 + j]) + xslack : -100000;
  }
  unsigned char tileLV[kMaxNTiles];
  double avg_pairs_V = 0.0;
  // a row of a sparse A (row_nnz nonzeros) contributes row_nnz terms to v_ij: the statistical tail bound of
  // the dropped pairs uses that contraction length (R8; the int32 capacity still uses n)
  const int64_t K_V = (P.row_nnz > 0 && P.row_nnz < n) ? P.row_nnz : n;
  int LV = tile_budgets(st.kA_split, kx, K_V, st.eA_max, c_col, tau_col, tileLV, &avg_pairs_V);
  if (P.L_V > 0) LV = P.L_V;
  LV = std::min(LV, st.kA_split + kx);
  const int kA = std::min(st.kA_split, LV - 1);
  rep.kA = kA;
  rep.L_V = LV;

  // ---- a2: X̂ → X̂^(1) + digits + r (exact), local columns; then the digit exchange (a11)
  double* X1 = ctx->ws<double>(S_X1, nnl);
  int8_t* xdig = ctx->ws<int8_t>(S_XDIG, static_cast<size_t>(7) * ld * n);
  int8_t* xdigT = ctx->ws<int8_t>(S_XDIGT, static_cast<size_t>(7) * ld * n);
  int32_t* g = ctx->ws<int32_t>(S_G, n);
  double* sh = ctx->ws<double>(S_SH, nl);
  double* sl = ctx->ws<double>(S_SL, nl);
  double* rh = ctx->ws<double>(S_RH, n);  // r_j of every column (all-gathered: the cluster branch reads them)
  double* rl = ctx->ws<double>(S_RL, n);
  OZR_ALLOC(X1); OZR_ALLOC(xdig); OZR_ALLOC(xdigT); OZR_ALLOC(g); OZR_ALLOC(sh); OZR_ALLOC(sl); OZR_ALLOC(rh);
  OZR_ALLOC(rl);
  ctx->mark("~");
  launch_x1_split(X, ldx, N, NL, beta, kx, w + col0, X1, n, xdig + col0 * ld, ld, ld * n, g + col0, sh, sl, rh + col0,
                  rl + col0, derr, s);
  OZR_CK(cudaGetLastError(), "x1 split");
  // a11: the digit planes, g and r of all columns — all-gathered on the side stream while the V product
  // (which needs only this rank's columns) runs; the main stream joins it before the transpose, i.e.
  // before any other collective is issued and before anything reads other ranks' columns
  if (ex) {
    cudaStream_t xs = ctx->xstream;
    OZR_CK(cudaEventRecord(ctx->xev[0], s), "event");
    OZR_CK(cudaStreamWaitEvent(xs, ctx->xev[0], 0), "wait");
    if (!ex->group_begin()) return fail(ctx, OZR_ERR_COMM, "%s", ex->err.c_str());
    for (int p = 0; p < kx; ++p) OZR_X(xgather_on(xdig + p * ld * n, static_cast<size_t>(nl * ld), xs));
    OZR_X(xgather_on(g, nl * sizeof(int32_t), xs));
    OZR_X(xgather_on(rh, nl * sizeof(double), xs));
    OZR_X(xgather_on(rl, nl * sizeof(double), xs));
    if (!ex->group_end(xs)) return fail(ctx, OZR_ERR_COMM, "%s", ex->err.c_str());
    OZR_CK(cudaEventRecord(ctx->xev[1], xs), "event");
  }
  ctx->mark("x1split");

  // ---- a3: P1  V = A·X̂^(1)_J  (Alg. 1 line 1, eq. mat_mul)
  std::vector<Group> gV = plan_groups(kA, kx, LV, n);
  PairTable pt;
  RecombPlan rp;
  if (!make_tables(gV, LV, n, pt, rp)) return fail(ctx, OZR_ERR_RANGE, "V plan too large");
  const bool tilesV = P.tile_budgets && P.L_V <= 0;
  if (tilesV) apply_tiles(pt, rp, tileLV, nl);
  rep.planes_V = avg_planes(rp, nl);
  size_t maxG = gV.size();
  int32_t* planes = ctx->ws<int32_t>(S_PLANES, maxG * nnl);
  OZR_ALLOC(planes);
  DigitOperand opA{reinterpret_cast<const int8_t*>(ctx->bufs[S_ADIG].p), ld, ld * n, st.kA_split};
  DigitOperand opXJ{xdig + col0 * ld, ld, ld * n, kx};  // local columns (B operand of V)
  DigitOperand opX{xdig, ld, ld * n, kx};               // all columns (A operand of W)
  // ---- a4-a6 (fused into the V bands): recombine V, λ̂, Res column maxima
  double* Vh = ctx->ws<double>(S_VH, nnl);
  double* Vl = ctx->ws<double>(S_VL, nnl);
  double* lam = ctx->ws<double>(S_LAM, n);
  int32_t* eR = ctx->ws<int32_t>(S_ER, nl);
  OZR_ALLOC(Vh); OZR_ALLOC(Vl); OZR_ALLOC(lam); OZR_ALLOC(eR);
  const int intmin = -(1 << 30);
  OZR_H2D(demax, &intmin, sizeof(int));
  const int32_t* aell = reinterpret_cast<const int32_t*>(ctx->bufs[S_AELL].p);
  const int scaleV = 8 * (st.kA_split + kx - LV);
  ctx->mark("~");
  OZR_X(run_banded(
      ctx, opA, opXJ, N, NL, N, pt, planes, 0,
      [&](int64_t c0, int64_t c1, int t0, int tma, cudaStream_t q) {
        launch_recombine_V(planes + c0 * n, nnl, N, static_cast<int>(c1 - c0), shift_plan(rp, t0), aell,
                           g + col0 + c0, scaleV, X1 + c0 * n, n, sh + c0, sl + c0, Vh + c0 * n, Vl + c0 * n, n,
                           lam + col0 + c0, eR + c0, demax, q, tma, lambda + col0 + c0);
      },
      [&](cudaStream_t q) {
        // the digit transpose (A operand of X̂Ẽ) needs every column's digits: after the exchange on P ranks
        if (ex) cudaStreamWaitEvent(q, ctx->xev[1], 0);
        launch_transpose_i8(xdig, ld, ld * n, xdigT, ld, ld * n, N, N, kx, q);
      }));
  ctx->mark("gemmV+recombV");
  // join the digit exchange before any other collective (λ̂ below) and before reading other ranks' digits
  if (ex) OZR_CK(cudaStreamWaitEvent(s, ctx->xev[1], 0), "wait exchange");
  // optional: R = I − X̂^(1)ᵀX̂^(1) (the R/S form's first product) to θ_W·δ' absolute
  double* nR2 = nullptr;
  if (P.form_R) {
    const int LG = std::min(choose_L(kx, kx, n, cmax + xslack, cmax + xslack, 0.5 * P.theta_W * delta_p), 2 * kx);
    std::vector<Group> gG = plan_groups(kx, kx, LG, n);
    PairTable ptG;
    RecombPlan rpG;
    if (!make_tables(gG, LG, n, ptG, rpG)) return fail(ctx, OZR_ERR_RANGE, "R plan too large");
    int32_t* planesG = ctx->ws<int32_t>(S_GPLANES, gG.size() * nnl);
    double* Rm = ctx->ws<double>(S_RMAT, nnl);
    nR2 = ctx->ws<double>(S_NR2, n);
    OZR_ALLOC(planesG); OZR_ALLOC(Rm); OZR_ALLOC(nR2);
    OZR_X(run_gemm(ctx, opX, opXJ, N, NL, N, ptG, planesG, 3));
    launch_form_R(planesG, nnl, N, NL, rpG, g, 8 * (2 * kx - LG), static_cast<int>(col0), rh, rl, Rm, n, nR2 + col0, s);
    OZR_CK(cudaGetLastError(), "form R");
    rep.pairs_G = count_pairs(gG);
    ops += 2.0 * n * n * nl * rep.pairs_G;
    ctx->last_R = Rm;
    ctx->last_R_n = n;
    ctx->last_R_nl = nl;
    ctx->mark("gemmG+R");
  }
  const double pV = tilesV ? avg_pairs_V : static_cast<double>(count_pairs(gV));
  rep.pairs_V = static_cast<int>(std::lround(pV));
  ops += 2.0 * n * n * nl * pV;

  OZR_X(xgather(lam, nl * sizeof(double)));
  int eRmax = 0;
  std::vector<double> hlam_new(n);
  std::vector<int> eR_col(nl);
  OZR_D2H(hlam_new.data(), lam, n * sizeof(double));
  OZR_D2H(eR_col.data(), eR, nl * sizeof(int32_t));
  // one synchronisation for λ̂, the Res exponents and their maximum; the digit transpose (A operand of
  // X̂Ẽ, after the exchange) runs meanwhile
  OZR_X(scalars({demax}, &eRmax));
  LamStats ls_new = lam_stats(hlam_new);
  const double gap_new0 = ls_new.gap0;
  if (!(gap_new0 > 0.0) && P.cluster_mode == 0) {  // name the offending pair (PAPER.md:333 assumes none)
    int pa = -1, pb = -1;
    equal_pair(hlam_new, &pa, &pb);
    return fail(ctx, OZR_ERR_DEGENERATE, "equal Rayleigh quotients λ̂_%d = λ̂_%d (gap = 0) with the cluster branch off",
                pa, pb);
  }
  const double gap_new = (gap_new0 > 0.0) ? gap_new0 : ls_new.gap_pos;
  if (eRmax == intmin) eRmax = -1074;

  // ---- a6: Res digits (k_R from the accuracy W needs, R8)
  const double gapW = std::min(gap, gap_new);
  const double tauW = P.theta_W * delta_p * gapW;
  // the fixed-slice plan (params.fixed_k) splits every operand into exactly k slices
  const int kR = P.fixed_k > 0 ? std::min(P.fixed_k, kMaxDigits)
                               : digits_for(eRmax, static_cast<int>(std::floor(std::log2(tauW / 2.0))));
  int8_t* rdig = ctx->ws<int8_t>(S_RDIG, static_cast<size_t>(kMaxDigits) * ld * nl);
  int32_t* rell = ctx->ws<int32_t>(S_RELL, nl);
  OZR_ALLOC(rdig); OZR_ALLOC(rell);
  ctx->mark("~");
  launch_split_res(Vh, Vl, n, X1, n, lam + col0, N, NL, kR, eR, rdig, ld, ld * nl, rell, s);
  OZR_CK(cudaGetLastError(), "split Res");
  ctx->mark("splitRes");

  // ---- a7: P3  W_{:,J} = X̂^(1)ᵀ Res_J  (Alg. 1 line 4)
  std::vector<double>& gaps_new = ls_new.colgap;
  for (double& x : gaps_new)
    if (!(x > 0.0)) x = gap_new;
  for (int64_t j = 0; j < nl; ++j) {
    tau_col[j] = 0.5 * P.theta_W * delta_p * (P.tile_budgets ? std::min(gaps_prev[col0 + j], gaps_new[col0 + j]) : gapW);
    if (eR_col[j] < -1000) eR_col[j] = -100000;
  }
  unsigned char tileLW[kMaxNTiles];
  double avg_pairs_W = 0.0;
  int LW = tile_budgets(kx, kR, n, cmax + xslack, eR_col, tau_col, tileLW, &avg_pairs_W);
  if (P.L_W > 0) LW = P.L_W;
  LW = std::min(LW, kx + kR);
  std::vector<Group> gW = plan_groups(kx, kR, LW, n);
  if (!make_tables(gW, LW, n, pt, rp)) return fail(ctx, OZR_ERR_RANGE, "W plan too large");
  const bool tilesW = P.tile_budgets && P.L_W <= 0;
  if (tilesW) apply_tiles(pt, rp, tileLW, nl);
  rep.planes_W = avg_planes(rp, nl);
  if (gW.size() > maxG) {
    maxG = gW.size();
    planes = ctx->ws<int32_t>(S_PLANES, maxG * nnl);
    OZR_ALLOC(planes);
  }
  DigitOperand opR{rdig, ld, ld * nl, kR};
  rep.kR = kR;
  rep.L_W = LW;
  const double pW = tilesW ? avg_pairs_W : static_cast<double>(count_pairs(gW));
  rep.pairs_W = static_cast<int>(std::lround(pW));
  ops += 2.0 * n * n * nl * pW;

  // ---- a8 (fused into the W bands): Ẽ (Alg. 1 line 5), Ẽ' = diag(2^g) Ẽ
  double* Ep = ctx->ws<double>(S_EP, nnl);
  double* nrm2 = ctx->ws<double>(S_NRM2, n);
  OZR_ALLOC(Ep); OZR_ALLOC(nrm2);
  OZR_H2D(demax, &intmin, sizeof(int));
  int* uf = ctx->ws<int>(S_EDGES, n);
  int* ecount = ctx->ws<int>(S_ECOUNT, 4);
  OZR_ALLOC(uf); OZR_ALLOC(ecount);
  OZR_CK(cudaMemsetAsync(ecount, 0, sizeof(int), s), "memset");
  if (P.cluster_mode) launch_iota(uf, N, s);
  const EdgeOut eo{P.cluster_mode, P.kappa, uf, ecount};
  double* nW2 = P.form_R ? ctx->ws<double>(S_NW2, n) : nullptr;
  if (P.form_R) OZR_ALLOC(nW2);
  const int scaleW = 8 * (kx + kR - LW);
  ctx->mark("~");
  OZR_X(run_banded(ctx, opX, opR, N, NL, N, pt, planes, 1,
                   [&](int64_t c0, int64_t c1, int t0, int tma, cudaStream_t q) {
                     launch_recombine_E(planes + c0 * n, nnl, N, static_cast<int>(c1 - c0), shift_plan(rp, t0), g,
                                        rell + c0, scaleW, rh + col0 + c0, lam, g, static_cast<int>(col0 + c0),
                                        Ep + c0 * n, n, nrm2 + col0 + c0, demax, eR + c0, derr, eo,
                                        nW2 ? nW2 + col0 + c0 : nullptr, q, tma);
                   }));
  ctx->mark("gemmW+recombE");
  int eEmax = 0, nedges = 0;
  std::vector<int> eE_col(nl);
  OZR_D2H(eE_col.data(), eR, nl * sizeof(int32_t));
  {
    int o2[2];
    OZR_X(scalars({demax, ecount}, o2));
    eEmax = o2[0];
    nedges = o2[1];
  }
  ctx->last_members.clear();
  ctx->last_offsets.assign(1, 0);
  int cluster_launches = P.cluster_mode ? 1 : 0;  // k_iota
  if (P.cluster_mode && nedges > 0) {
    // ---- a8 cluster branch (R13): unresolved groups → Rayleigh–Ritz sub-solve (cluster.cu)
    cluster_launches += 1;  // k_uf_flatten
    launch_uf_flatten(uf, N, s);
    std::vector<int> root(n);
    if (NP == 1) {
      OZR_D2H(root.data(), uf, n * sizeof(int));
      OZR_CK(cudaStreamSynchronize(s), "sync");
      ctx->flush();
    } else {  // every rank's partition of the pairs it saw → one union on the host, in rank order
      int* ufall = ctx->ws<int>(S_UFALL, static_cast<size_t>(NP) * n);
      OZR_ALLOC(ufall);
      OZR_CK(cudaMemcpyAsync(ufall + RK * n, uf, n * sizeof(int), cudaMemcpyDeviceToDevice, s), "D2D");
      OZR_X(xgather(ufall, n * sizeof(int)));
      std::vector<int> lab(static_cast<size_t>(NP) * n);
      OZR_D2H(lab.data(), ufall, lab.size() * sizeof(int));
      OZR_CK(cudaStreamSynchronize(s), "sync");
      ctx->flush();
      for (int64_t i = 0; i < n; ++i) root[i] = static_cast<int>(i);
      auto find = [&](int a) {
        while (root[a] != a) {
          root[a] = root[root[a]];
          a = root[a];
        }
        return a;
      };
      for (int r = 0; r < NP; ++r)
        for (int64_t i = 0; i < n; ++i) {
          const int a = find(static_cast<int>(i)), b = find(lab[r * n + i]);
          if (a != b) root[std::max(a, b)] = std::min(a, b);
        }
      for (int64_t i = 0; i < n; ++i) root[i] = find(static_cast<int>(i));
    }
    std::vector<int>& mem = ctx->last_members;
    std::vector<int>& off = ctx->last_offsets;
    unresolved_groups(n, root, hlam_new, mem, off);
    const int ng = static_cast<int>(off.size()) - 1;
    if (ng > 0) {
      int mmax = 0;
      std::vector<int> gm(ng), gsq(ng + 1, 0), grp_of(n, -1), pos_of(n, 0);
      std::vector<double> mu(ng);
      std::vector<int4> tiles, tiles_tc;
      // groups from this size on get their Gram block G_JJ = X̂_JᵀX̂_J from the INT8 slice GEMM (all digit
      // pairs: the same exact integers as k_cluster_dot's int64 sums, rounded once) — OZR_TC_GRAM=0 disables
      const bool tc_on = !(getenv("OZR_TC_GRAM") && getenv("OZR_TC_GRAM")[0] == '0');
      const int tc_min = tc_on ? std::max(2, P.dense_cluster) : (1 << 30);
      for (int q = 0; q < ng; ++q) {
        const int m = off[q + 1] - off[q];
        gm[q] = m;
        mmax = std::max(mmax, m);
        gsq[q + 1] = gsq[q] + m * m;
        double sm = 0.0;
        for (int a = 0; a < m; ++a) {
          const int j = mem[off[q] + a];
          sm = sm + hlam_new[j];
          grp_of[j] = q;
          pos_of[j] = a;
        }
        mu[q] = sm / m;
        std::vector<int4>& tl = (m >= tc_min) ? tiles_tc : tiles;
        for (int a0 = 0; a0 < m; a0 += 16)
          for (int b0 = 0; b0 < m; b0 += 16) tl.push_back(make_int4(q, a0, b0, m));
      }
      const int ntiles_dot = static_cast<int>(tiles.size());  // small groups first: k_cluster_dot covers them
      tiles.insert(tiles.end(), tiles_tc.begin(), tiles_tc.end());
      if (mmax > P.max_cluster)
        return fail(ctx, OZR_ERR_RANGE, "unresolved group of %d columns exceeds max_cluster = %d", mmax, P.max_cluster);
      const int nmem = off[ng];
      // one packed int upload: tiles | off | gsq | gm | mem | grp_of | pos_of | sweeps
      std::vector<int> pk;
      pk.reserve(tiles.size() * 4 + 3 * ng + 2 + nmem + 2 * n + ng + 8);
      for (const int4& t : tiles) { pk.push_back(t.x); pk.push_back(t.y); pk.push_back(t.z); pk.push_back(t.w); }
      const size_t o_off = pk.size(); pk.insert(pk.end(), off.begin(), off.end());
      const size_t o_gsq = pk.size(); pk.insert(pk.end(), gsq.begin(), gsq.end());
      const size_t o_gm = pk.size(); pk.insert(pk.end(), gm.begin(), gm.end());
      const size_t o_mem = pk.size(); pk.insert(pk.end(), mem.begin(), mem.end());
      const size_t o_grp = pk.size(); pk.insert(pk.end(), grp_of.begin(), grp_of.end());
      const size_t o_pos = pk.size(); pk.insert(pk.end(), pos_of.begin(), pos_of.end());
      const size_t o_sw = pk.size(); pk.resize(pk.size() + ng);
      int* dpk = ctx->ws<int>(S_CINT, pk.size());
      double* dmu = ctx->ws<double>(S_CDBL, ng);
      const size_t sq = static_cast<size_t>(gsq[ng]);
      double* cM = ctx->ws<double>(S_CM, sq);
      double* cR = ctx->ws<double>(S_CR, sq);
      double* cK = ctx->ws<double>(S_CK, sq);
      double* cV = ctx->ws<double>(S_CV, sq);
      double* cZ = ctx->ws<double>(S_CZ, sq);
      double* cT = ctx->ws<double>(S_CT, static_cast<size_t>(nmem) * n);
      OZR_ALLOC(dpk); OZR_ALLOC(dmu); OZR_ALLOC(cM); OZR_ALLOC(cR); OZR_ALLOC(cK); OZR_ALLOC(cV); OZR_ALLOC(cZ);
      OZR_ALLOC(cT);
      OZR_H2D(dpk, pk.data(), pk.size() * sizeof(int));
      OZR_H2D(dmu, mu.data(), ng * sizeof(double));
      ClusterLaunch L{};
      L.ngroups = ng;
      L.nmembers = nmem;
      L.mmax = mmax;
      L.ntiles = static_cast<int>(tiles.size());
      L.ntiles_dot = ntiles_dot;
      L.Gbuf = cK;  // K is only written by the solve, after the build has read G
      L.rows = N;
      L.col0 = static_cast<int>(col0);
      L.ncols = NL;
      L.tiles = reinterpret_cast<const int4*>(dpk);
      L.goff = dpk + o_off;
      L.gsq = dpk + o_gsq;
      L.gm = dpk + o_gm;
      L.mem = dpk + o_mem;
      L.grp_of = dpk + o_grp;
      L.pos_of = dpk + o_pos;
      L.mu = dmu;
      L.xdig = xdig;
      L.ldd = ld;
      L.pstride = ld * n;
      L.kx = kx;
      L.gexp = g;
      L.r_hi = rh;
      L.r_lo = rl;
      L.wplanes = planes;
      L.wpstride = nnl;
      L.rpW = &rp;
      L.ellR = rell;
      L.scale8 = 8 * (kx + kR - LW);
      L.lam = lam;
      L.Mbuf = cM; L.Rbuf = cR; L.Kbuf = cK; L.Vbuf = cV; L.Zbuf = cZ; L.T = cT;
      L.sweeps = dpk + o_sw;
      L.Ep = Ep;
      L.lde = n;
      L.nrm2 = nrm2;
      L.eE_col = eR;
      L.eE_max = demax;
      L.nsplit = cluster_dot_splits(std::max(1, L.ntiles_dot), N);
      L.part = ctx->ws<unsigned long long>(S_CPART, static_cast<size_t>(std::max(1, L.ntiles_dot)) * L.nsplit * 512);
      OZR_ALLOC(L.part);
      L.hgm = gm.data();
      L.coop_scratch = ctx->ws<double>(S_CSCR, 5 * static_cast<size_t>(mmax) + 8);
      L.coop_flags = ctx->ws<int>(S_CFLAG, 128);
      OZR_ALLOC(L.coop_scratch); OZR_ALLOC(L.coop_flags);
      L.dense_min = P.dense_cluster > 0 ? P.dense_cluster : (1 << 30);
      L.err = derr;
      // (1) M_JJ columns owned by this rank, (2) all-reduce → full M on every rank, (3) Jacobi (replicated),
      // (4) T = Ẽ'[:, J] owned columns, all-reduce, (5) apply + column statistics on owned columns
      // tensor-core Gram of the large groups: gather their digit columns, all-pairs slice GEMM, exact
      // recombination rounded once to fp64 (scaled by 2^{g_a + g_b}), into G = cK at the group's offset
      for (int q = 0; q < ng; ++q) {
        if (gm[q] < tc_min) continue;
        const int m = gm[q];
        int8_t* xg = ctx->ws<int8_t>(S_CXG, static_cast<size_t>(kx) * ld * m);
        int32_t* gJ = ctx->ws<int32_t>(S_CGJ, m);
        OZR_ALLOC(xg); OZR_ALLOC(gJ);
        launch_gather_digit_cols(xdig, ld, ld * n, kx, dpk + o_mem + off[q], m, xg, ld * m, g, gJ, s);
        const int LG = 2 * kx;
        std::vector<Group> gG = plan_groups(kx, kx, LG, n);
        PairTable ptG;
        RecombPlan rpG;
        if (!make_tables(gG, LG, n, ptG, rpG)) return fail(ctx, OZR_ERR_RANGE, "Gram plan too large");
        const size_t mm = static_cast<size_t>(m) * m;
        int32_t* gplanes = ctx->ws<int32_t>(S_CGP, gG.size() * mm);
        int* cnt = ctx->ws<int>(S_GCNT, 4);
        OZR_ALLOC(gplanes); OZR_ALLOC(cnt);
        const DigitOperand opG{xg, ld, ld * m, kx};
        OZR_CK(launch_gemm_i8(opG, opG, m, m, N, ptG, gplanes, static_cast<int64_t>(mm), m, s, cnt), "Gram GEMM");
        launch_recombine_dd(gplanes, static_cast<long long>(mm), m, m, rpG, gJ, gJ, 0, cK + gsq[q], nullptr, m, s);
        OZR_CK(cudaGetLastError(), "Gram recombination");
        cluster_launches += 3;
      }
      OZR_CK(launch_cluster_build(L, s), "cluster build");
      OZR_X(xsum(cM, sq));
      OZR_CK(launch_cluster_solve(L, s), "cluster solve");
      // dense sub-solve of the large groups (dense_eig.cu): K = C·sym(M)·C and Z = C·Y with C = I + R/2 as
      // FP64-accurate INT8 slice products (R = R_JJ is symmetric: no transpose for its split)
      double* dP = nullptr;
      double* dth = nullptr;
      if (mmax >= L.dense_min) {
        dP = ctx->ws<double>(S_DP, static_cast<size_t>(mmax) * mmax);
        dth = ctx->ws<double>(S_DTH, mmax);
        OZR_ALLOC(dP); OZR_ALLOC(dth);
      }
      for (int q = 0; q < ng; ++q) {
        if (gm[q] < L.dense_min) continue;
        const int m = gm[q];
        const long long mm = static_cast<long long>(m) * m;
        double* M = cM + gsq[q];
        double* R = cR + gsq[q];
        double* K = cK + gsq[q];
        double* V = cV + gsq[q];
        double* Z = cZ + gsq[q];
        launch_dense_sym(m, M, V, s);                                   // V = K0 = (M + Mᵀ)/2
        OZR_X(oz_dgemm(ctx, m, m, m, R, m, true, V, m, dP, m, derr));    // P = R·K0
        launch_dense_axpy(mm, V, 0.5, dP, K, s);                        // K = K0 + ½R·K0 = C·K0
        OZR_X(oz_dgemm(ctx, m, m, m, K, m, false, R, m, dP, m, derr));   // P = K·R
        launch_dense_axpy(mm, K, 0.5, dP, V, s);                        // V = C·K0·C
        launch_dense_sym(m, V, K, s);                                   // K = sym(V)
        {
          std::string why;
          const SyevGemm gemm = [&](int M2, int N2, int K2, const double* A2, int lda2, bool at, const double* B2,
                                    int ldb2, double* C2, int ldc2) {
            return oz_dgemm(ctx, M2, N2, K2, A2, lda2, at, B2, ldb2, C2, ldc2, derr) == OZR_OK ? 0 : 1;
          };
          const int rc = dense_syev(ctx->syev, m, K, dth, K, gemm, kSyevBigGemm, s, &why);
          if (rc != 0) return fail(ctx, rc == 8 ? OZR_ERR_NOMEM : OZR_ERR_CUDA, "dense cluster eigensolver: %s", why.c_str());
        }
        launch_dense_sign(m, K, dth, mu[q], dpk + o_mem + off[q], lam, nullptr, derr, s);  // K = Y
        OZR_X(oz_dgemm(ctx, m, m, m, R, m, true, K, m, dP, m, derr));    // P = R·Y
        launch_dense_axpy(mm, K, 0.5, dP, Z, s);                        // Z = Y + ½R·Y = C·Y
        OZR_CK(cudaGetLastError(), "dense cluster solve");
        cluster_launches += 18;
      }
      OZR_X(xsum(cT, static_cast<size_t>(nmem) * n));
      OZR_CK(launch_cluster_apply(L, s), "cluster apply");
      if (mmax >= L.dense_min) {
        double* TZ = ctx->ws<double>(S_DTZ, static_cast<size_t>(n) * mmax);
        OZR_ALLOC(TZ);
        for (int q = 0; q < ng; ++q) {
          if (gm[q] < L.dense_min) continue;
          const int m = gm[q];
          OZR_X(oz_dgemm(ctx, n, m, m, cT + static_cast<size_t>(off[q]) * n, n, false, cZ + gsq[q], m, TZ, n, derr));
          launch_dense_scatter(TZ, N, m, dpk + o_mem + off[q], q, dpk + o_grp, dpk + o_pos, cZ + gsq[q], g, Ep, n,
                               static_cast<int>(col0), NL, s);
          cluster_launches += 6;
        }
      }
      OZR_CK(launch_cluster_colstats(L, s), "cluster column statistics");
      ctx->mark("cluster");
      cluster_launches += 6;
      OZR_D2H(hlam_new.data(), lam, n * sizeof(double));
      OZR_D2H(eE_col.data(), eR, nl * sizeof(int32_t));
      OZR_X(scalars({demax}, &eEmax));
      rep.n_clusters = ng;
      rep.max_cluster = mmax;
    }
  }
  if (eEmax == intmin) eEmax = -1074;
  // g_j = ⌈log2 w_j⌉ + β − 53 (k_x1_split; ⌈log2 0⌉ := 0), so its minimum is known on the host
  int gmin = 100000;
  for (double x : hw) gmin = std::min(gmin, (x != 0.0 ? ceil_log2_host(x) : 0) + beta - 53);

  // ---- a9: P4  U_J = X̂^(1) Ẽ_{:,J} = Q Ẽ'_{:,J} ; X̂_J ← RN(X̂^(1)_J + U_J)  (Alg. 1 line 6)
  const double tauU = P.theta_U * delta_p;
  const int kE = P.fixed_k > 0 ? std::min(P.fixed_k, kMaxDigits)
                               : digits_for(eEmax, static_cast<int>(std::floor(std::log2(tauU / 2.0))) + gmin);
  ctx->mark("~");
  launch_split_fixed(Ep, nullptr, n, N, NL, kE, rdig, ld, ld * nl, rell, derr, s);
  OZR_CK(cudaGetLastError(), "split E");
  ctx->mark("splitE");
  const int SX = 8 * (kx - 1) + 6;
  // R8b for X̂Ẽ: uniform accuracy θ_U·δ', but columns with small corrections need fewer pairs
  for (int64_t j = 0; j < nl; ++j) tau_col[j] = tauU / 2.0;
  unsigned char tileLU[kMaxNTiles];
  double avg_pairs_U = 0.0;
  int LU = tile_budgets(kx, kE, n, SX, eE_col, tau_col, tileLU, &avg_pairs_U);
  if (P.L_U > 0) LU = P.L_U;
  LU = std::min(LU, kx + kE);
  std::vector<Group> gU = plan_groups(kx, kE, LU, n);
  if (!make_tables(gU, LU, n, pt, rp)) return fail(ctx, OZR_ERR_RANGE, "U plan too large");
  const bool tilesU = P.tile_budgets && P.L_U <= 0;
  if (tilesU) apply_tiles(pt, rp, tileLU, nl);
  rep.planes_U = avg_planes(rp, nl);
  if (gU.size() > maxG) {
    maxG = gU.size();
    planes = ctx->ws<int32_t>(S_PLANES, maxG * nnl);
    OZR_ALLOC(planes);
  }
  DigitOperand opQ{xdigT, ld, ld * n, kx};
  DigitOperand opE{rdig, ld, ld * nl, kE};
  rep.kE = kE;
  rep.L_U = LU;
  const double pU = tilesU ? avg_pairs_U : static_cast<double>(count_pairs(gU));
  rep.pairs_U = static_cast<int>(std::lround(pU));
  ops += 2.0 * n * n * nl * pU;
  double* nu2 = ctx->ws<double>(S_NU2, n);
  OZR_ALLOC(nu2);
  const int scaleU = 8 * (kx + kE - LU);
  ctx->mark("~");
  OZR_X(run_banded(ctx, opQ, opE, N, NL, N, pt, planes, 2,
                   [&](int64_t c0, int64_t c1, int t0, int tma, cudaStream_t q) {
                     launch_final(planes + c0 * n, nnl, N, static_cast<int>(c1 - c0), shift_plan(rp, t0), rell + c0,
                                  scaleU, X1 + c0 * n, n, X + c0 * ldx, ldx, nu2 + col0 + c0, wnext + col0 + c0, q, tma);
                   }));
  ctx->mark("gemmU+final");
  OZR_X(xgather(nu2, nl * sizeof(double)));
  OZR_X(xgather(nrm2, nl * sizeof(double)));
  std::vector<double> hR2, hW2;
  if (P.form_R) {
    OZR_X(xgather(nR2, nl * sizeof(double)));
    OZR_X(xgather(nW2, nl * sizeof(double)));
    hR2.resize(n);
    hW2.resize(n);
    OZR_D2H(hR2.data(), nR2, n * sizeof(double));
    OZR_D2H(hW2.data(), nW2, n * sizeof(double));
  }
  OZR_CK(cudaMemcpyAsync(lambda, lam, n * sizeof(double), cudaMemcpyDeviceToDevice, s), "copy lambda");
  cudaEventRecord(ctx->ev[1], s);
  std::vector<double> hnu(n), hnrm(n);
  OZR_D2H(hnu.data(), nu2, n * sizeof(double));
  OZR_D2H(hnrm.data(), nrm2, n * sizeof(double));
  OZR_X(scalars({}, nullptr));
  ctx->mark("~end");
  double nu = 0.0, ne = 0.0;
  for (int64_t j = 0; j < n; ++j) {
    nu += hnu[j];
    ne += hnrm[j];
  }
  float tot = 0.f;
  cudaEventElapsedTime(&tot, ctx->ev[0], ctx->ev[1]);
  for (int q = 0; q < (P.form_R ? 4 : 3); ++q) {
    float t = 0.f;
    cudaEventElapsedTime(&t, ctx->ev[2 + 2 * q], ctx->ev[3 + 2 * q]);
    gemm_ms += t;
  }
  if (P.form_R) {
    double r2 = 0.0, w2 = 0.0;
    for (int64_t j = 0; j < n; ++j) {
      r2 += hR2[j];
      w2 += hW2[j];
    }
    rep.normR_fro = std::sqrt(r2);
    rep.normW_fro = std::sqrt(w2);
    rep.omega_oa = 2.0 * (rep.normW_fro + 2.0 * maxlam * rep.normR_fro);
  }
  st.have_w = true;
  rep.net_update = std::sqrt(nu);
  rep.normE_fro = std::sqrt(ne);
  if (rep.n_clusters > 0) ls_new = lam_stats(hlam_new);  // the sub-solve changed λ̂_J
  const double maxlam_new = ls_new.maxabs;
  const double gap_out = ls_new.gap_pos;
  rep.predicted_error = rep.net_update * rep.net_update * maxlam_new / (static_cast<double>(n) * gap_out);
  if (ex) {  // report the global pair budgets (each rank planned its own column tiles)
    int hv[3] = {rep.L_V, rep.L_W, rep.L_U}, gv[3];
    OZR_H2D(scal + 4 * NP, hv, sizeof hv);
    int* d = scal + 4 * NP;
    OZR_X(scalars({d, d + 1, d + 2}, gv));
    rep.L_V = gv[0];
    rep.L_W = gv[1];
    rep.L_U = gv[2];
    rep.kA = std::min(st.kA_split, rep.L_V - 1);
  }
  rep.ms_total = tot;
  rep.ms_gemm = gemm_ms;
  rep.int8_ops = ops;
  rep.exchanges = nexch;
  ctx->dump();
  // kernels of this sweep: [colmax] x1_split transpose split_res split_E, and per column band of each of the
  // three products its GEMM and its recombination (recombine_V / recombine_E / final)
  rep.launches = (fresh_w ? 1 : 0) + 4 + 6 * band_count(NL) + cluster_launches + (new_A ? 2 : 0) + (P.form_R ? 2 : 0) +
                 ctx->staged_launches;
#undef OZR_X
  return OZR_OK;
}

constexpr double kCertSafety = 1.15;  // power-iteration / bf16-GEMM slack of the estimate (R12)
constexpr double kContract = 1.0 / 8;  // an estimate that fell by less than this sits at the truncation floor

// a10 (R12): the a-posteriori forward-error estimate of the sweep just completed, from its own Ẽ (certify.cu):
//   est = sqrt(‖D‖₂² + (2u)²) + ‖Ẽ‖_F‖D‖_F + 2u‖(λ̂_i ẽ_ij/(λ̂_j − λ̂_i))_{i≠j}‖_F,   D = −(E − Ẽ) to second order:
//   D_ij = q_ij/(λ̂_j − λ̂_i) − (Ẽ²)_ij (i ≠ j), D_jj = −(Ẽ²)_jj − ½‖ẽ_j‖², Q = ẼᵀC, c_kj = (λ̂_k − λ̂_j)ẽ_kj
// (oracle/refine.second_order_defect), plus the fp64 rounding of X̂_new, an allowance for the third-order
// terms and the defect from the fp64 rounding of the λ̂ in Ẽ's denominators (certify.cu header). ‖D‖₂ comes from its Frobenius norm when that already certifies, from the power iteration otherwise —
// except when even the lower bound max_j ‖D_{:,j}‖ exceeds 16δ: then the upper bound (Frobenius) is reported,
// which no decision of the driver can tell from the exact value.
// Reads the sweep's Ẽ' (S_EP), g (S_G) and λ̂ (S_LAM); writes rep.cert, cert_q, cert_frob, cert_iters.
ozr_status certify(ozr_ctx ctx, Exchange* ex, int64_t n, double delta, ozr_step_report& rep) {
  const int NP = ex ? ex->P : 1, RK = ex ? ex->rank : 0;
  const int64_t nl = n / NP, col0 = RK * nl, nnl = n * nl;
  const int N = static_cast<int>(n), NL = static_cast<int>(nl);
  cudaStream_t s = ctx->stream;
  const int64_t ldb = round16(n);  // bf16 elements per column (32-byte aligned columns)
  const double* Ep = static_cast<const double*>(ctx->bufs[S_EP].p);
  const int32_t* g = static_cast<const int32_t*>(ctx->bufs[S_G].p);
  const double* lam = static_cast<const double*>(ctx->bufs[S_LAM].p);
  uint16_t* Eb = ctx->ws<uint16_t>(S_CEB, static_cast<size_t>(ldb) * n);
  uint16_t* EbT = ctx->ws<uint16_t>(S_CEBT, static_cast<size_t>(ldb) * n);
  uint16_t* Cb = ctx->ws<uint16_t>(S_CCB, static_cast<size_t>(ldb) * nl);
  int32_t* sE = ctx->ws<int32_t>(S_CSE, n);
  int32_t* sC = ctx->ws<int32_t>(S_CSC, nl);
  int32_t* rE = ctx->ws<int32_t>(S_CRE, n);
  double* esq = ctx->ws<double>(S_CESQ, 2 * n);  // Σ_i ẽ_ij² per column, then the eigenvalue-rounding sums
  double* rsq = esq + n;
  double* dsq = ctx->ws<double>(S_CDSQ, n);
  int* flag = ctx->ws<int>(S_CFLG, 4);
  float* Q = reinterpret_cast<float*>(ctx->ws<int32_t>(S_PLANES, nnl));  // the slice planes are dead by now
  float* Dw = reinterpret_cast<float*>(ctx->ws<double>(S_VH, nnl));     // so is V (2·nnl floats: D (bf16), then P)
  __nv_bfloat16* D = reinterpret_cast<__nv_bfloat16*>(Dw);
  float* Pm = Dw + nnl;
  int* cnt = ctx->ws<int>(S_GCNT, 4);
  double* z = ctx->ws<double>(S_PI_Z, nl);
  double* v = ctx->ws<double>(S_PI_V, nl);
  double* y = ctx->ws<double>(S_PI_Y, n);
  double* part = ctx->ws<double>(S_PI_P, static_cast<size_t>(cert_pi_chunks()) * n);
  double* sc = ctx->ws<double>(S_PI_S, 2);
  OZR_ALLOC(Eb); OZR_ALLOC(EbT); OZR_ALLOC(Cb); OZR_ALLOC(sE); OZR_ALLOC(sC); OZR_ALLOC(rE); OZR_ALLOC(esq);
  OZR_ALLOC(dsq); OZR_ALLOC(flag); OZR_ALLOC(Q); OZR_ALLOC(Dw); OZR_ALLOC(cnt); OZR_ALLOC(z); OZR_ALLOC(v); OZR_ALLOC(y);
  OZR_ALLOC(part); OZR_ALLOC(sc);
  auto gather = [&](void* base, size_t bytes) -> ozr_status {
    if (ex && !ex->allgather(base, bytes, s)) return fail(ctx, OZR_ERR_COMM, "all-gather: %s", ex->err.c_str());
    return OZR_OK;
  };
  auto allsum = [&](double* b, size_t c) -> ozr_status {
    if (ex && !ex->allreduce_sum(b, c, s)) return fail(ctx, OZR_ERR_COMM, "all-reduce: %s", ex->err.c_str());
    return OZR_OK;
  };
  ozr_status e;
  OZR_CK(cudaMemsetAsync(flag, 0, sizeof(int), s), "memset");
  launch_cert_prep(Ep, n, N, NL, g, lam, static_cast<int>(col0), Eb, Cb, ldb, sE, sC, esq + col0, rsq + col0, s);
  if ((e = gather(Eb, static_cast<size_t>(nl) * ldb * 2)) != OZR_OK) return e;  // all columns: the A operand
  if ((e = gather(sE, nl * sizeof(int32_t))) != OZR_OK) return e;
  if ((e = gather(esq, nl * sizeof(double))) != OZR_OK) return e;
  if ((e = gather(rsq, nl * sizeof(double))) != OZR_OK) return e;
  launch_cert_rowT(Eb, ldb, N, N, sE, rE, EbT, s);
  PairTable pt;
  memset(&pt, 0, sizeof pt);
  pt.ngroups = 1;
  pt.first[1] = 1;
  pt.diag[0] = 2;
  const DigitOperand opE{reinterpret_cast<const int8_t*>(Eb), 2 * ldb, 2 * ldb * n, 1};
  const DigitOperand opC{reinterpret_cast<const int8_t*>(Cb), 2 * ldb, 2 * ldb * nl, 1};
  const DigitOperand opET{reinterpret_cast<const int8_t*>(EbT), 2 * ldb, 2 * ldb * n, 1};
  const DigitOperand opEJ{reinterpret_cast<const int8_t*>(Eb + col0 * ldb), 2 * ldb, 2 * ldb * nl, 1};
  OZR_CK(launch_gemm_i8(opE, opC, N, NL, 2 * N, pt, reinterpret_cast<int32_t*>(Q), nnl, n, s, cnt, 1, 1),
         "certificate GEMM Q (bf16)");
  OZR_CK(launch_gemm_i8(opET, opEJ, N, NL, 2 * N, pt, reinterpret_cast<int32_t*>(Pm), nnl, n, s, cnt, 1, 1),
         "certificate GEMM E^2 (bf16)");
  launch_cert_delta(Q, Pm, n, N, NL, sE, sC, rE, esq, lam, static_cast<int>(col0), D, dsq + col0, flag, s);
  OZR_CK(cudaGetLastError(), "certificate");
  if ((e = gather(dsq, nl * sizeof(double))) != OZR_OK) return e;
  std::vector<double> hesq(2 * n), hdsq(n);
  int hflag = 0;
  ctx->pend.clear();
  ctx->hst_off = 0;
  OZR_D2H(hesq.data(), esq, 2 * n * sizeof(double));
  OZR_D2H(hdsq.data(), dsq, n * sizeof(double));
  OZR_D2H(&hflag, flag, sizeof(int));
  OZR_CK(cudaStreamSynchronize(s), "sync");
  ctx->flush();
  rep.cert_iters = 0;
  if (hflag) {  // equal estimates outside a group: no certificate
    rep.cert = rep.cert_q = rep.cert_frob = INFINITY;
    return OZR_OK;
  }
  double e2 = 0.0, d2 = 0.0, dmax = 0.0, r2 = 0.0;
  for (int64_t j = 0; j < n; ++j) {
    e2 += hesq[j];
    r2 += hesq[n + j];
    d2 += hdsq[j];
    dmax = std::max(dmax, hdsq[j]);
  }
  // quad: the third-order allowance ‖Ẽ‖_F‖D‖_F plus the defect Ẽ carries from the fp64 rounding of the λ̂ it
  // divided by, ≤ 2u·sqrt(Σ_{i≠j} (λ̂_i ẽ_ij/(λ̂_j − λ̂_i))²) (certify.cu header)
  const double frob = std::sqrt(d2), quad = std::sqrt(e2) * frob + 2.0 * kU * std::sqrt(r2), rnd = 2.0 * kU;
  rep.cert_frob = frob;
  const double upper = std::sqrt(frob * frob + rnd * rnd) + quad;
  if (upper * kCertSafety <= delta || std::sqrt(dmax) + quad > 16.0 * delta) {
    rep.cert = upper;
    rep.cert_q = frob;
    return OZR_OK;
  }
  // ‖D‖₂ by Golub–Kahan–Lanczos bidiagonalization (D column-partitioned: D·v all-reduced, Dᵀu local), no
  // reorthogonalisation (the largest Ritz value still converges to σ_max from below): β₀u₀ = Dv₀,
  // α_j v_{j+1} = Dᵀu_j − β_j v_j, β_{j+1}u_{j+1} = Dv_{j+1} − α_j u_j; σ_max of the upper bidiagonal B
  // (diag β, super α) from the largest eigenvalue of BᵀB by bisection. Checked every 4 steps from step 8 on:
  // stop when it moved by ≤ 1e-3 relative (at most 40 steps).
  constexpr int kLzMax = 40;
  double* lz = ctx->ws<double>(S_PI_LZ, 2 * (kLzMax + 2));  // bsq[0..], asq[0..]
  double* u = ctx->ws<double>(S_PI_U, n);
  double* t = ctx->ws<double>(S_PI_T, nl);
  OZR_ALLOC(lz); OZR_ALLOC(u); OZR_ALLOC(t);
  double* bsq = lz;
  double* asq = lz + kLzMax + 2;
  auto sigma_max = [](const std::vector<double>& b2, const std::vector<double>& a2, int k) {
    // T = BᵀB: T_ii = β_i² + α_{i−1}², T_{i,i+1} = α_i β_i (squared off-diagonal α_i²β_i² for the Sturm count)
    std::vector<double> dg(k), off2(k, 0.0);
    double hi = 0.0;
    for (int i = 0; i < k; ++i) {
      dg[i] = b2[i] + (i > 0 ? a2[i - 1] : 0.0);
      if (i + 1 < k) off2[i] = a2[i] * b2[i];
    }
    for (int i = 0; i < k; ++i)
      hi = std::max(hi, dg[i] + (i > 0 ? std::sqrt(off2[i - 1]) : 0.0) + (i + 1 < k ? std::sqrt(off2[i]) : 0.0));
    double lo = 0.0;
    for (int it = 0; it < 200 && hi - lo > 1e-14 * hi; ++it) {
      const double x = 0.5 * (lo + hi);
      int cnt = 0;  // eigenvalues of T greater than x (Sturm sequence of T − xI)
      double q = dg[0] - x;
      if (q > 0) ++cnt;
      for (int i = 1; i < k; ++i) {
        q = dg[i] - x - off2[i - 1] / (q != 0.0 ? q : 1e-300);
        if (q > 0) ++cnt;
      }
      if (cnt >= 1) lo = x; else hi = x;
    }
    return std::sqrt(0.5 * (lo + hi));
  };
  launch_normalize(v, nullptr, NL, nullptr, static_cast<int>(col0), s);  // deterministic start
  launch_sumsq(v, NL, sc, s);
  if ((e = allsum(sc, 1)) != OZR_OK) return e;
  launch_normalize(z, v, NL, sc, 0, s);  // z = v₀ (unit)
  launch_pi_dz(D, N, NL, z, part, y, s);
  if ((e = allsum(y, n)) != OZR_OK) return e;
  launch_sumsq(y, N, bsq, s);
  launch_normalize(u, y, N, bsq, 0, s);
  double sig = 0.0, prev = -1.0;
  int k = 0;
  std::vector<double> hb(kLzMax + 2), ha(kLzMax + 2);
  while (k < kLzMax) {
    const int kn = std::min(kLzMax, k < 8 ? 8 : k + 4);
    for (; k < kn; ++k) {
      launch_pi_dty(D, N, NL, u, t, s);                 // t = Dᵀu_k
      launch_lz_axpy(z, t, NL, bsq + k, s);             // z ← t − β_k v_k (z holds v_k)
      launch_sumsq(z, NL, asq + k, s);
      if ((e = allsum(asq + k, 1)) != OZR_OK) return e;
      launch_normalize(z, z, NL, asq + k, 0, s);        // v_{k+1}
      launch_pi_dz(D, N, NL, z, part, y, s);            // y = D v_{k+1}
      if ((e = allsum(y, n)) != OZR_OK) return e;
      launch_lz_axpy(u, y, N, asq + k, s);              // u ← y − α_k u_k
      launch_sumsq(u, N, bsq + k + 1, s);
      launch_normalize(u, u, N, bsq + k + 1, 0, s);     // u_{k+1}
    }
    OZR_CK(cudaGetLastError(), "Lanczos");
    ctx->pend.clear();
    ctx->hst_off = 0;
    OZR_D2H(hb.data(), bsq, (k + 1) * sizeof(double));
    OZR_D2H(ha.data(), asq, k * sizeof(double));
    OZR_CK(cudaStreamSynchronize(s), "sync");
    ctx->flush();
    sig = sigma_max(hb, ha, k);
    if (prev > 0.0 && std::fabs(sig - prev) <= 1e-3 * sig) break;
    prev = sig;
  }
  rep.cert_iters = k;
  rep.cert_q = sig;
  rep.cert = std::sqrt(sig * sig + rnd * rnd) + quad;
  return OZR_OK;
}

ozr_status check_ctx(ozr_ctx ctx) {
  if (!ctx) return OZR_ERR_ARG;
  OZR_CK(cudaSetDevice(ctx->device), "cudaSetDevice");
  return OZR_OK;
}

// Guard-band mode: every workspace buffer's guard band still holds the pattern (after all queued work)
ozr_status guard_check(ozr_ctx ctx, ozr_status st) {
  if (!ctx || !ctx->guard) return st;
  cudaStreamSynchronize(ctx->stream);
  int bad = ctx->guard_bad;
  for (size_t i = 0; i < ctx->bufs.size() && bad < 0; ++i)
    if (ctx->bufs[i].p && !ctx->guard_ok(ctx->bufs[i])) bad = static_cast<int>(i);
  if (bad >= 0) return fail(ctx, OZR_ERR_CUDA, "guard band of workspace slot %d overwritten", bad);
  return st;
}

}  // namespace

// ================================================================ C ABI
extern "C" {

const char* ozr_version(void) { return "ozr 0.1 (sm_100a, tcgen05 kind::i8)"; }

ozr_status ozr_create(ozr_ctx* out, int device, void* stream, int64_t n_max) {
  (void)n_max;
  if (!out) return OZR_ERR_ARG;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    cudaGetLastError();
    return OZR_ERR_CUDA;
  }
  if (cudaSetDevice(device) != cudaSuccess) return OZR_ERR_CUDA;
  ozr_ctx c = new ozr_ctx_s();
  c->device = device;
  c->stream = static_cast<cudaStream_t>(stream);
  for (int i = 0; i < 10; ++i) cudaEventCreate(&c->ev[i]);
  cudaStreamCreateWithFlags(&c->xstream, cudaStreamNonBlocking);
  cudaEventCreateWithFlags(&c->ev_sync, cudaEventDisableTiming);
  for (int i = 0; i < 2; ++i) cudaEventCreateWithFlags(&c->xev[i], cudaEventDisableTiming);
  {
    int lo = 0, hi = 0;  // the recombination bands get the higher priority: their CTAs fill the SM room the
    cudaDeviceGetStreamPriorityRange(&lo, &hi);  // persistent GEMM leaves as soon as they are ready
    (void)lo;
    cudaStreamCreateWithPriority(&c->rstream, cudaStreamNonBlocking, hi);
  }
  for (int i = 0; i < kMaxBands + 2; ++i) cudaEventCreateWithFlags(&c->bev[i], cudaEventDisableTiming);
  c->events = true;
  const char* tr = getenv("OZR_TRACE");
  c->trace = tr && tr[0] == '1';
  const char* gd = getenv("OZR_GUARD");
  c->guard = gd && gd[0] == '1';
  *out = c;
  return OZR_OK;
}

void ozr_destroy(ozr_ctx ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (auto& b : ctx->bufs)
    if (b.p) cudaFree(b.p);
  if (ctx->events)
    for (int i = 0; i < 10; ++i) cudaEventDestroy(ctx->ev[i]);
  for (int i = 0; i < 2; ++i) cudaEventDestroy(ctx->xev[i]);
  if (ctx->xstream) cudaStreamDestroy(ctx->xstream);
  if (ctx->rstream) {
    cudaStreamSynchronize(ctx->rstream);
    cudaStreamDestroy(ctx->rstream);
  }
  for (int i = 0; i < kMaxBands + 2; ++i) cudaEventDestroy(ctx->bev[i]);
  if (ctx->ev_sync) cudaEventDestroy(ctx->ev_sync);
  if (ctx->hst) cudaFreeHost(ctx->hst);
  delete ctx;
}

const char* ozr_last_error(ozr_ctx ctx) { return ctx ? ctx->err.c_str() : "null context"; }

void ozr_params_default(ozr_params* p) {
  if (!p) return;
  memset(p, 0, sizeof *p);
  p->delta = 1e-12;
  p->theta = 4.0;  // R11: the O(δ) result lands at or below δ
  p->beta_mode = 0;
  p->xi = 0.0;
  p->beta_override = 0;
  p->truncate = 1;
  p->max_sweeps = 6;
  p->kA_split = 15;
  p->theta_V = 1.0 / 16;
  p->theta_W = 1.0 / 16;
  p->theta_U = 1.0 / 16;
  p->cluster_mode = 1;
  p->tile_budgets = 1;
  p->kappa = 0x1p-10;
  p->max_cluster = 16384;
  p->form_R = 0;
  p->dense_cluster = 64;  // measured (tools/dev/dense_thr.py): c2's 67-column group 2.33 -> 1.71 ms per sweep; c4 unchanged
  p->max_escalations = 2;
  p->certify = 1;
  p->fixed_k = 0;
}

ozr_status ozr_split(ozr_ctx ctx, const double* M, const double* M_lo, int64_t rows, int64_t cols, int64_t ldm,
                     int axis, int mode, int k_or_beta, int8_t* digits, int64_t ldd, int64_t plane_stride,
                     int32_t* lsb_exp, double* x1_out, int64_t ldx1, int* k_out) {
  ozr_status st = check_ctx(ctx);
  if (st != OZR_OK) return st;
  if (!M || !digits || !lsb_exp || rows <= 0 || cols <= 0 || ldm < rows || (ldd % 16) || (plane_stride % 16))
    return fail(ctx, OZR_ERR_ARG, "ozr_split: bad argument");
  if (rows > (int64_t(1) << 31) || cols > (int64_t(1) << 31)) return fail(ctx, OZR_ERR_ARG, "ozr_split: too large");
  cudaStream_t s = ctx->stream;
  int* derr = ctx->ws<int>(S_ERR, 4);
  OZR_ALLOC(derr);
  OZR_CK(cudaMemsetAsync(derr, 0, sizeof(int), s), "memset");
  if (mode == OZR_SPLIT_X1) {
    if (axis != OZR_COLWISE || M_lo) return fail(ctx, OZR_ERR_ARG, "ozr_split: X1 mode is COLWISE, fp64 only");
    const int beta = k_or_beta;
    if (beta < kBetaMin || beta > kBetaMax) return fail(ctx, OZR_ERR_RANGE, "ozr_split: beta must be in [2, 52]");
    if (ldd < rows || plane_stride < ldd * cols) return fail(ctx, OZR_ERR_ARG, "ozr_split: digit layout too small");
    const int kx = kx_for_beta(beta);
    double* w = ctx->ws<double>(S_W, cols);
    double* X1 = x1_out ? x1_out : ctx->ws<double>(S_TMP1, rows * cols);
    const int64_t ld1 = x1_out ? ldx1 : rows;
    double* tmp = ctx->ws<double>(S_TMP2, 4 * cols);
    OZR_ALLOC(w); OZR_ALLOC(X1); OZR_ALLOC(tmp);
    if (x1_out && ldx1 < rows) return fail(ctx, OZR_ERR_ARG, "ozr_split: ldx1 < rows");
    launch_colmax(M, ldm, static_cast<int>(rows), static_cast<int>(cols), w, derr, s);
    launch_x1_split(M, ldm, static_cast<int>(rows), static_cast<int>(cols), beta, kx, w, X1, ld1, digits, ldd,
                    plane_stride, lsb_exp, tmp, tmp + cols, tmp + 2 * cols, tmp + 3 * cols, derr, s);
    OZR_CK(cudaGetLastError(), "ozr_split");
    if (k_out) *k_out = kx;
    // a zero column is legal for a split (ERR_DEGENERATE only matters to the refinement)
    int h = 0;
    OZR_CK(cudaMemcpyAsync(&h, derr, sizeof(int), cudaMemcpyDeviceToHost, s), "D2H");
    OZR_CK(cudaStreamSynchronize(s), "sync");
    if (h & ERR_NONFINITE) return fail(ctx, OZR_ERR_NONFINITE, "non-finite value in M");
    if (h & ERR_RANGE) return fail(ctx, OZR_ERR_RANGE, "exponent range exceeded");
    return OZR_OK;
  }
  if (mode != OZR_SPLIT_FIXED) return fail(ctx, OZR_ERR_ARG, "ozr_split: bad mode");
  const int k = k_or_beta;
  if (k < 1 || k > kMaxDigits) return fail(ctx, OZR_ERR_RANGE, "ozr_split: k must be in [1, 15]");
  const double* src = M;
  const double* srcl = M_lo;
  int64_t r = rows, c = cols, lds = ldm;
  if (axis == OZR_ROWWISE) {
    double* T = ctx->ws<double>(S_TMP1, rows * cols);
    OZR_ALLOC(T);
    launch_transpose_f64(M, ldm, T, cols, static_cast<int>(rows), static_cast<int>(cols), s);
    src = T;
    if (M_lo) {
      double* Tl = ctx->ws<double>(S_TMP2, rows * cols);
      OZR_ALLOC(Tl);
      launch_transpose_f64(M_lo, ldm, Tl, cols, static_cast<int>(rows), static_cast<int>(cols), s);
      srcl = Tl;
    }
    r = cols;
    c = rows;
    lds = cols;
  } else if (axis != OZR_COLWISE) {
    return fail(ctx, OZR_ERR_ARG, "ozr_split: bad axis");
  }
  if (ldd < r || plane_stride < ldd * c) return fail(ctx, OZR_ERR_ARG, "ozr_split: digit layout too small");
  launch_split_fixed(src, srcl, lds, static_cast<int>(r), static_cast<int>(c), k, digits, ldd, plane_stride, lsb_exp,
                     derr, s);
  OZR_CK(cudaGetLastError(), "ozr_split");
  if (k_out) *k_out = k;
  return read_err(ctx, derr);
}

ozr_status ozr_syev(ozr_ctx ctx, int64_t m, const double* K, int64_t ldk, double* theta, double* Y, int64_t ldy) {
  ozr_status st = check_ctx(ctx);
  if (st != OZR_OK) return st;
  if (!K || !theta || !Y || m < 1 || ldk < m || ldy < m || m > 32768) return fail(ctx, OZR_ERR_ARG, "ozr_syev: bad argument");
  cudaStream_t s = ctx->stream;
  const size_t mm = static_cast<size_t>(m) * m;
  double* Kw = ctx->ws<double>(S_DP, mm);  // working copy (destroyed by the tridiagonalisation)
  double* Yw = ctx->ws<double>(S_DTZ, mm);
  int* derr = ctx->ws<int>(S_ERR, 4);
  OZR_ALLOC(Kw); OZR_ALLOC(Yw); OZR_ALLOC(derr);
  OZR_CK(cudaMemsetAsync(derr, 0, sizeof(int), s), "memset");
  OZR_CK(cudaMemcpy2DAsync(Kw, m * sizeof(double), K, ldk * sizeof(double), m * sizeof(double), m,
                           cudaMemcpyDeviceToDevice, s), "copy K");
  std::string why;
  const SyevGemm gemm = [&](int M2, int N2, int K2, const double* A2, int lda2, bool at, const double* B2, int ldb2,
                            double* C2, int ldc2) {
    return oz_dgemm(ctx, M2, N2, K2, A2, lda2, at, B2, ldb2, C2, ldc2, derr) == OZR_OK ? 0 : 1;
  };
  const int rc = dense_syev(ctx->syev, static_cast<int>(m), Kw, theta, Yw, gemm, kSyevBigGemm, s, &why);
  if (rc != 0) return fail(ctx, rc == 8 ? OZR_ERR_NOMEM : OZR_ERR_CUDA, "ozr_syev: %s", why.c_str());
  OZR_CK(cudaMemcpy2DAsync(Y, ldy * sizeof(double), Yw, m * sizeof(double), m * sizeof(double), m,
                           cudaMemcpyDeviceToDevice, s), "copy Y");
  OZR_CK(cudaStreamSynchronize(s), "sync");
  return guard_check(ctx, OZR_OK);
}

ozr_status ozr_syev_tridiag(ozr_ctx ctx, int64_t m, double* K, int64_t ldk, double* d, double* e, double* tau) {
  ozr_status st = check_ctx(ctx);
  if (st != OZR_OK) return st;
  if (!K || !d || !e || !tau || m < 1 || ldk != m || m > 32768) return fail(ctx, OZR_ERR_ARG, "ozr_syev_tridiag: bad argument");
  ozr::SyevDebug dbg;
  dbg.d_out = d;
  dbg.e_out = e;
  dbg.tau_out = tau;
  std::string why;
  const int rc = dense_syev(ctx->syev, static_cast<int>(m), K, nullptr, nullptr, nullptr, 0, ctx->stream, &why, &dbg);
  if (rc != 0) return fail(ctx, rc == 8 ? OZR_ERR_NOMEM : OZR_ERR_CUDA, "ozr_syev_tridiag: %s", why.c_str());
  return OZR_OK;
}

ozr_status ozr_syev_tridiag_eig(ozr_ctx ctx, int64_t m, const double* d, const double* e, double* theta, double* Y,
                                int64_t ldy) {
  ozr_status st = check_ctx(ctx);
  if (st != OZR_OK) return st;
  if (!d || !e || !theta || !Y || m < 1 || ldy != m || m > 32768) return fail(ctx, OZR_ERR_ARG, "ozr_syev_tridiag_eig: bad argument");
  int* derr = ctx->ws<int>(S_ERR, 4);
  OZR_ALLOC(derr);
  ozr::SyevDebug dbg;
  dbg.d_in = d;
  dbg.e_in = e;
  std::string why;
  const SyevGemm gemm = [&](int M2, int N2, int K2, const double* A2, int lda2, bool at, const double* B2, int ldb2,
                            double* C2, int ldc2) {
    return oz_dgemm(ctx, M2, N2, K2, A2, lda2, at, B2, ldb2, C2, ldc2, derr) == OZR_OK ? 0 : 1;
  };
  const int rc = dense_syev(ctx->syev, static_cast<int>(m), nullptr, theta, Y, gemm, kSyevBigGemm, ctx->stream, &why, &dbg);
  if (rc != 0) return fail(ctx, rc == 8 ? OZR_ERR_NOMEM : OZR_ERR_CUDA, "ozr_syev_tridiag_eig: %s", why.c_str());
  return OZR_OK;
}

ozr_status ozr_last_R(ozr_ctx ctx, double* R, int64_t ldr) {
  if (!ctx || !R || !ctx->last_R || ldr < ctx->last_R_n) return OZR_ERR_ARG;
  OZR_CK(cudaMemcpy2DAsync(R, ldr * sizeof(double), ctx->last_R, ctx->last_R_n * sizeof(double),
                           ctx->last_R_n * sizeof(double), ctx->last_R_nl, cudaMemcpyDeviceToDevice, ctx->stream),
         "copy R");
  OZR_CK(cudaStreamSynchronize(ctx->stream), "sync");
  return OZR_OK;
}

ozr_status ozr_last_clusters(ozr_ctx ctx, int* members, int max_members, int* offsets, int max_groups, int* ngroups) {
  if (!ctx) return OZR_ERR_ARG;
  const int ng = static_cast<int>(ctx->last_offsets.size()) - 1;
  if (ngroups) *ngroups = ng;
  if (offsets && max_groups >= ng)
    for (int q = 0; q <= ng; ++q) offsets[q] = ctx->last_offsets[q];
  const int nm = ctx->last_offsets[ng];
  if (max_groups < ng || max_members < nm || (nm > 0 && (!members || !offsets))) return OZR_ERR_RANGE;
  for (int q = 0; q < nm; ++q) members[q] = ctx->last_members[q];
  return OZR_OK;
}

ozr_status ozr_gemm_plan(int64_t k, int kA, int kB, int L, int* ngroups, int* group_diag, int* group_npairs,
                         int max_groups) {
  if (k <= 0 || kA < 1 || kB < 1 || kA > kMaxDigits || kB > kMaxDigits) return OZR_ERR_RANGE;
  if (L <= 0) L = kA + kB;
  std::vector<Group> gs = plan_groups(kA, kB, L, k);
  if (ngroups) *ngroups = static_cast<int>(gs.size());
  for (int i = 0; i < static_cast<int>(gs.size()) && i < max_groups; ++i) {
    if (group_diag) group_diag[i] = gs[i].d;
    if (group_npairs) group_npairs[i] = static_cast<int>(gs[i].pairs.size());
  }
  return OZR_OK;
}

ozr_status ozr_gemm(ozr_ctx ctx, int64_t m, int64_t n, int64_t k, const double* A, int64_t lda, const double* B,
                    int64_t ldb, int kA, int kB, int L, double* C_hi, double* C_lo, int64_t ldc, int32_t* planes_out,
                    int64_t plane_stride, int* ngroups_out) {
  ozr_status st = check_ctx(ctx);
  if (st != OZR_OK) return st;
  if (!A || !B || !C_hi || m <= 0 || n <= 0 || k <= 0 || lda < m || ldb < k || ldc < m)
    return fail(ctx, OZR_ERR_ARG, "ozr_gemm: bad argument");
  if (kA < 1 || kB < 1 || kA > kMaxDigits || kB > kMaxDigits) return fail(ctx, OZR_ERR_RANGE, "ozr_gemm: kA/kB");
  if (k * 16384 > 2147483647LL) return fail(ctx, OZR_ERR_RANGE, "ozr_gemm: k too large for exact int32 slices");
  if (L <= 0) L = kA + kB;
  cudaStream_t s = ctx->stream;
  const int64_t ldk = round16(k);
  int8_t* da = ctx->ws<int8_t>(S_RDIG, static_cast<size_t>(kA) * ldk * m);
  int8_t* db = ctx->ws<int8_t>(S_XDIG, static_cast<size_t>(kB) * ldk * n);
  int32_t* ea = ctx->ws<int32_t>(S_AELL, m);
  int32_t* eb = ctx->ws<int32_t>(S_BELL, n);
  OZR_ALLOC(da); OZR_ALLOC(db); OZR_ALLOC(ea); OZR_ALLOC(eb);
  st = ozr_split(ctx, A, nullptr, m, k, lda, OZR_ROWWISE, OZR_SPLIT_FIXED, kA, da, ldk, ldk * m, ea, nullptr, 0,
                 nullptr);
  if (st != OZR_OK) return st;
  st = ozr_split(ctx, B, nullptr, k, n, ldb, OZR_COLWISE, OZR_SPLIT_FIXED, kB, db, ldk, ldk * n, eb, nullptr, 0,
                 nullptr);
  if (st != OZR_OK) return st;
  std::vector<Group> gs = plan_groups(kA, kB, L, k);
  PairTable pt;
  RecombPlan rp;
  if (!make_tables(gs, L, k, pt, rp)) return fail(ctx, OZR_ERR_RANGE, "ozr_gemm: plan too large");
  if (ngroups_out) *ngroups_out = pt.ngroups;
  const int64_t mn = m * n;
  int32_t* planes = planes_out;
  int64_t ps = plane_stride;
  if (!planes) {
    planes = ctx->ws<int32_t>(S_PLANES, static_cast<size_t>(pt.ngroups) * mn);
    OZR_ALLOC(planes);
    ps = mn;
  } else if (plane_stride < mn) {
    return fail(ctx, OZR_ERR_ARG, "ozr_gemm: plane_stride < m*n");
  }
  DigitOperand oa{da, ldk, ldk * m, kA}, ob{db, ldk, ldk * n, kB};
  int* cnt = ctx->ws<int>(S_GCNT, 4);
  OZR_ALLOC(cnt);
  OZR_CK(launch_gemm_i8(oa, ob, static_cast<int>(m), static_cast<int>(n), static_cast<int>(k), pt, planes, ps, m, s, cnt),
         "slice GEMM");
  launch_recombine_dd(planes, ps, static_cast<int>(m), static_cast<int>(n), rp, ea, eb, 8 * (kA + kB - L), C_hi, C_lo,
                      ldc, s);
  OZR_CK(cudaGetLastError(), "recombine");
  return guard_check(ctx, OZR_OK);
}

// The Hermitian extension of one sweep (R18; include/ozr.h): Algorithm 1 with
// conjugate transposes, every complex product one real INT8 slice product of the stacked form (herm.cu), the
// β of §4.1 and the accuracy-driven digit budgets of the real sweep (R8) with uniform (per-product) budgets.
ozr_status ozr_refine_step_herm(ozr_ctx ctx, const double* Ar, const double* Ai, int64_t n, int64_t lda, double* Xr,
                                double* Xi, int64_t ldx, double* lambda, const ozr_params* params,
                                ozr_step_report* report) {
  ozr_status st = check_ctx(ctx);
  if (st != OZR_OK) return st;
  if (!Ar || !Ai || !Xr || !Xi || !lambda || !params || n < 2 || lda < n || ldx < n)
    return fail(ctx, OZR_ERR_ARG, "ozr_refine_step_herm: bad argument");
  if (2 * n * 16384 > 2147483647LL) return fail(ctx, OZR_ERR_RANGE, "ozr_refine_step_herm: n too large");
  const ozr_params P = *params;
  if (P.delta <= 0.0) return fail(ctx, OZR_ERR_ARG, "ozr_refine_step_herm: delta <= 0");
  ozr_step_report rep;
  memset(&rep, 0, sizeof rep);
  cudaStream_t s = ctx->stream;
  cudaEventRecord(ctx->ev[0], s);
  const int N = static_cast<int>(n), N2 = 2 * N;
  const int64_t n2 = 2 * n;
  const int64_t ld2 = round16(n2);
  int* derr = ctx->ws<int>(S_ERR, 4);
  double* Xs = ctx->ws<double>(S_HXS, static_cast<size_t>(n2) * n);
  double* X1 = ctx->ws<double>(S_HX1, static_cast<size_t>(n2) * n);
  int8_t* xd = ctx->ws<int8_t>(S_HXD, static_cast<size_t>(7) * ld2 * n);
  int32_t* g = ctx->ws<int32_t>(S_HG, n);
  double* sh = ctx->ws<double>(S_HSH, n);
  double* sl = ctx->ws<double>(S_HSL, n);
  double* rh = ctx->ws<double>(S_HRH, n);
  double* rl = ctx->ws<double>(S_HRL, n);
  double* v1 = ctx->ws<double>(S_HV1, n2);
  double* v2 = ctx->ws<double>(S_HV2, n2);
  double* lamn = ctx->ws<double>(S_HV3, n);
  double* nrm = ctx->ws<double>(S_HV4, n);
  OZR_ALLOC(derr); OZR_ALLOC(Xs); OZR_ALLOC(X1); OZR_ALLOC(xd); OZR_ALLOC(g); OZR_ALLOC(sh); OZR_ALLOC(sl);
  OZR_ALLOC(rh); OZR_ALLOC(rl); OZR_ALLOC(v1); OZR_ALLOC(v2); OZR_ALLOC(lamn); OZR_ALLOC(nrm);
  OZR_CK(cudaMemsetAsync(derr, 0, 4 * sizeof(int), s), "memset");
  auto rd = [&](void* h, const void* d, size_t bytes) -> ozr_status {
    OZR_CK(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s), "D2H");
    OZR_CK(cudaStreamSynchronize(s), "sync");
    return OZR_OK;
  };
  auto errs = [&]() -> ozr_status {
    int h = 0;
    ozr_status e = rd(&h, derr, sizeof(int));
    if (e != OZR_OK) return e;
    return err_bits(ctx, h);
  };
  auto emax_of = [&](const std::vector<double>& v) {
    int e = -100000;
    for (double x : v)
      if (x != 0.0) e = std::max(e, ceil_log2_host(x));
    return e;
  };
  ozr_status e;
  // ---- X̂s = [Xr; Xi] (2n x n), w_j = max over the stacked column, λ̂ statistics, β (§4.1)
  OZR_CK(cudaMemcpy2DAsync(Xs, n2 * sizeof(double), Xr, ldx * sizeof(double), n * sizeof(double), n,
                           cudaMemcpyDeviceToDevice, s), "stack X");
  OZR_CK(cudaMemcpy2DAsync(Xs + n, n2 * sizeof(double), Xi, ldx * sizeof(double), n * sizeof(double), n,
                           cudaMemcpyDeviceToDevice, s), "stack X");
  launch_colmax(Xs, n2, N2, N, v1, derr, s);
  std::vector<double> hw(n), hlam(n);
  if ((e = rd(hw.data(), v1, n * sizeof(double))) != OZR_OK) return e;
  if ((e = rd(hlam.data(), lambda, n * sizeof(double))) != OZR_OK) return e;
  if ((e = errs()) != OZR_OK) return e;
  for (double x : hlam)
    if (!std::isfinite(x)) return fail(ctx, OZR_ERR_NONFINITE, "non-finite lambda");
  const double delta_p = P.delta / (P.theta > 0 ? P.theta : 1.0);
  LamStats ls = lam_stats(hlam);
  if (!(ls.gap0 > 0.0)) return fail(ctx, OZR_ERR_DEGENERATE, "equal eigenvalue estimates (PAPER.md:333)");
  const double ssum = sum_pow2_2c(hw);
  if (ssum == 0.0 || ls.maxabs == 0.0) return fail(ctx, OZR_ERR_DEGENERATE, "zero X or zero spectrum");
  const int beta_raw = (P.beta_override > 0) ? P.beta_override
                                             : choose_beta(n, delta_p, P.beta_mode, P.xi, ls.gap0, ls.maxabs, ssum, 0);
  const int beta = std::min(std::max(beta_raw, kBetaMin), kBetaMax);
  const int kx = kx_for_beta(beta);
  int cmax = -100000, gmin = 100000;
  for (double x : hw) {
    const int c = x != 0.0 ? ceil_log2_host(x) : 0;
    if (x != 0.0) cmax = std::max(cmax, c);
    gmin = std::min(gmin, c + beta - 53);
  }
  rep.beta = beta;
  rep.beta_raw = beta_raw;
  rep.alpha = alpha_dense(n, beta);
  rep.kX = kx;
  rep.gap_min = ls.gap0;
  rep.max_abs_lambda = ls.maxabs;
  // ---- X̂ → X̂^(1) (τ trick on both parts with the column's τ_j), g_j, x̂_jᴴx̂_j and r_j exactly
  launch_x1_split(Xs, n2, N2, N, beta, kx, v1, X1, n2, xd, ld2, ld2 * n, g, sh, sl, rh, rl, derr, s);
  OZR_CK(cudaGetLastError(), "x1 split");
  // ---- V̂ = M_A·X̂s^(1) (Alg. 1 line 1), M_A = [[Ar, −Ai], [Ai, Ar]] (real symmetric, 2n x 2n)
  double* MA = ctx->ws<double>(S_HMA, static_cast<size_t>(n2) * n2);
  double* Vh = ctx->ws<double>(S_HVH, static_cast<size_t>(n2) * n);
  double* Vl = ctx->ws<double>(S_HVL, static_cast<size_t>(n2) * n);
  OZR_ALLOC(MA); OZR_ALLOC(Vh); OZR_ALLOC(Vl);
  launch_herm_embed(Ar, Ai, lda, N, MA, n2, s);
  launch_colmax(MA, n2, N2, N2, v2, derr, s);
  std::vector<double> hv(n2);
  if ((e = rd(hv.data(), v2, n2 * sizeof(double))) != OZR_OK) return e;
  if ((e = errs()) != OZR_OK) return e;
  const int eA = emax_of(hv);
  const double tauV = P.theta_V * delta_p * ls.gap0;
  int LV = P.L_V > 0 ? P.L_V : choose_L(kMaxDigits, kx, n2, eA, cmax, tauV);
  LV = std::min(LV, kMaxDigits + kx);
  const int kA = std::min(kMaxDigits, LV - 1);
  rep.kA = kA;
  rep.L_V = LV;
  int pV = 0, pW = 0, pU = 0;
  if ((e = herm_product(ctx, n2, n, n2, MA, n2, true, X1, n2, kA, kx, LV, Vh, Vl, n2, derr, &pV)) != OZR_OK) return e;
  // ---- λ̂ (line 3), R̂ and JR̂ (line 4's right operand)
  double* R2 = ctx->ws<double>(S_HR2, static_cast<size_t>(n2) * n2);
  OZR_ALLOC(R2);
  launch_herm_lam_res(Vh, Vl, n2, X1, n2, sh, sl, N, lamn, R2, n2, v1, s);
  OZR_CK(cudaGetLastError(), "lambda / residual");
  std::vector<double> hrm(n), hlam_new(n);
  if ((e = rd(hrm.data(), v1, n * sizeof(double))) != OZR_OK) return e;
  if ((e = rd(hlam_new.data(), lamn, n * sizeof(double))) != OZR_OK) return e;
  if ((e = errs()) != OZR_OK) return e;
  LamStats ls_new = lam_stats(hlam_new);
  if (!(ls_new.gap0 > 0.0)) return fail(ctx, OZR_ERR_DEGENERATE, "equal Rayleigh quotients (PAPER.md:333)");
  // ---- W = X̂ᴴR = X̂sᵀ·[R̂, JR̂] (n x 2n: [Re W, Im W]) (line 4)
  const int eR = emax_of(hrm);
  const double tauW = P.theta_W * delta_p * std::min(ls.gap0, ls_new.gap0);
  const int kR = eR == -100000 ? 1 : digits_for(eR, static_cast<int>(std::floor(std::log2(tauW / 2.0))));
  int LW = P.L_W > 0 ? P.L_W : choose_L(kx, kR, n2, cmax, eR == -100000 ? -1074 : eR, tauW);
  LW = std::min(LW, kx + kR);
  rep.kR = kR;
  rep.L_W = LW;
  double* Wd = ctx->ws<double>(S_HW, static_cast<size_t>(n) * n2);
  OZR_ALLOC(Wd);
  if ((e = herm_product(ctx, n, n2, n2, X1, n2, true, R2, n2, kx, kR, LW, Wd, nullptr, n, derr, &pW)) != OZR_OK)
    return e;
  // ---- Ẽ (line 5) as the B operand of U, and Q (U's A operand)
  double* Bm = ctx->ws<double>(S_HB, static_cast<size_t>(n2) * n2);
  double* Q = ctx->ws<double>(S_HQ, static_cast<size_t>(n) * n2);
  OZR_ALLOC(Bm); OZR_ALLOC(Q);
  launch_herm_E(Wd, n, lamn, rh, g, N, Bm, n2, nrm, v1, derr, s);
  launch_herm_Q(X1, n2, g, N, Q, n, s);
  OZR_CK(cudaGetLastError(), "E / Q");
  std::vector<double> hem(n), hnrm(n);
  if ((e = rd(hem.data(), v1, n * sizeof(double))) != OZR_OK) return e;
  if ((e = rd(hnrm.data(), nrm, n * sizeof(double))) != OZR_OK) return e;
  if ((e = errs()) != OZR_OK) return e;
  double e2 = 0.0;
  for (double x : hnrm) e2 += x;
  rep.normE_fro = std::sqrt(e2);
  // ---- U = X̂^(1)Ẽ = Q·[E1, E2] (n x 2n: [Re U, Im U]), X̂ ← RN(X̂^(1) + U) (line 6)
  const double tauU = P.theta_U * delta_p;
  int eE = emax_of(hem);
  if (eE == -100000) eE = -1074;
  const int kE = digits_for(eE, static_cast<int>(std::floor(std::log2(tauU / 2.0))) + gmin);
  const int SX = 8 * (kx - 1) + 6;
  int LU = P.L_U > 0 ? P.L_U : choose_L(kx, kE, n2, SX, eE, tauU);
  LU = std::min(LU, kx + kE);
  rep.kE = kE;
  rep.L_U = LU;
  double* Uh = ctx->ws<double>(S_HUH, static_cast<size_t>(n) * n2);
  double* Ul = ctx->ws<double>(S_HUL, static_cast<size_t>(n) * n2);
  OZR_ALLOC(Uh); OZR_ALLOC(Ul);
  if ((e = herm_product(ctx, n, n2, n2, Q, n, false, Bm, n2, kx, kE, LU, Uh, Ul, n, derr, &pU)) != OZR_OK) return e;
  launch_herm_final(Uh, Ul, n, X1, n2, Xr, Xi, ldx, N, nrm, s);
  OZR_CK(cudaGetLastError(), "accsum");
  OZR_CK(cudaMemcpyAsync(lambda, lamn, n * sizeof(double), cudaMemcpyDeviceToDevice, s), "lambda");
  if ((e = rd(hnrm.data(), nrm, n * sizeof(double))) != OZR_OK) return e;
  if ((e = errs()) != OZR_OK) return e;
  double nu = 0.0;
  for (double x : hnrm) nu += x;
  rep.net_update = std::sqrt(nu);
  rep.pairs_V = pV;
  rep.pairs_W = pW;
  rep.pairs_U = pU;
  rep.int8_ops = 2.0 * static_cast<double>(n2) * n * n2 * pV + 2.0 * static_cast<double>(n) * n2 * n2 * (pW + pU);
  rep.sweep = 1;
  rep.theta = P.theta;
  rep.cert = -1.0;
  cudaEventRecord(ctx->ev[1], s);
  cudaEventSynchronize(ctx->ev[1]);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[1]);
  rep.ms_total = ms;
  if (report) *report = rep;
  return guard_check(ctx, OZR_OK);
}

struct ozr_comm_s {
  std::unique_ptr<ozr::Exchange> ex;
};

ozr_status ozr_comm_nccl_id(void* id128) {
  if (!id128) return OZR_ERR_ARG;
  std::string err;
  return nccl_unique_id(id128, err) ? OZR_OK : OZR_ERR_COMM;
}

ozr_status ozr_comm_create_nccl(ozr_comm* out, const void* id128, int nranks, int rank, int device) {
  if (!out || !id128 || nranks < 1 || rank < 0 || rank >= nranks) return OZR_ERR_ARG;
  *out = nullptr;
  if (cudaSetDevice(device) != cudaSuccess) return OZR_ERR_CUDA;
  std::string err;
  NcclExchange* ex = nccl_create(id128, nranks, rank, err);
  if (!ex) {
    fprintf(stderr, "ozr: %s\n", err.c_str());
    return OZR_ERR_COMM;
  }
  ozr_comm c = new ozr_comm_s();
  c->ex.reset(ex);
  *out = c;
  return OZR_OK;
}

ozr_status ozr_comm_create_host_group(ozr_comm* out, int nranks) {
  if (!out || nranks < 1) return OZR_ERR_ARG;
  auto grp = std::make_shared<HostGroup>(nranks);
  for (int r = 0; r < nranks; ++r) {
    HostExchange* ex = new HostExchange();
    ex->P = nranks;
    ex->rank = r;
    ex->g = grp;
    out[r] = new ozr_comm_s();
    out[r]->ex.reset(ex);
  }
  return OZR_OK;
}

void ozr_comm_destroy(ozr_comm comm) { delete comm; }
int ozr_comm_size(ozr_comm comm) { return comm ? comm->ex->P : 1; }
int ozr_comm_rank(ozr_comm comm) { return comm ? comm->ex->rank : 0; }

namespace {
// params.fixed_k: the prior work's fixed-slice plan as a digit plan
ozr_params effective_params(const ozr_params& in) {
  ozr_params P = in;
  if (P.fixed_k > 0) {
    P.truncate = 0;
    P.L_V = P.L_W = P.L_U = P.fixed_k + 1;
  }
  return P;
}

ozr_status check_refine_args(ozr_ctx ctx, ozr_comm comm, const double* A, int64_t n, int64_t lda, const double* X,
                             int64_t ldx, const double* lambda, const ozr_params* params) {
  ozr_status st = check_ctx(ctx);
  if (st != OZR_OK) return st;
  if (!A || !X || !lambda || !params || n < 2 || lda < n || ldx < n)
    return fail(ctx, OZR_ERR_ARG, "ozr_refine: bad argument");
  if (n > 65536) return fail(ctx, OZR_ERR_ARG, "ozr_refine: n too large");
  if (comm && (n % comm->ex->P != 0 || n / comm->ex->P < 1))
    return fail(ctx, OZR_ERR_ARG, "ozr_refine: n must be a multiple of the number of ranks");
  if (!(params->delta > kU)) return fail(ctx, OZR_ERR_RANGE, "delta must exceed u = 2^-53");
  if (params->kA_split < 2 || params->kA_split > kMaxDigits) return fail(ctx, OZR_ERR_RANGE, "kA_split");
  return OZR_OK;
}
}  // namespace

ozr_status ozr_refine_step_dist(ozr_ctx ctx, ozr_comm comm, const double* A, int64_t n, int64_t lda, double* X,
                                int64_t ldx, double* lambda, const ozr_params* params, ozr_step_report* report) {
  ozr_status st = check_refine_args(ctx, comm, A, n, lda, X, ldx, lambda, params);
  if (st != OZR_OK) return st;
  SweepState ss;
  ozr_step_report rep;
  const ozr_params P = effective_params(*params);
  st = sweep(ctx, comm ? comm->ex.get() : nullptr, A, n, lda, X, ldx, lambda, P, rep, ss);
  rep.sweep = 1;
  rep.theta = params->theta;
  rep.cert = -1.0;
  if (st == OZR_OK && params->certify >= 2 && rep.n_clusters == 0)
    st = certify(ctx, comm ? comm->ex.get() : nullptr, n, params->delta, rep);
  if (report) *report = rep;
  return guard_check(ctx, st);
}

// The driver (R12; the paper iterates a fixed number of times): after every sweep without
// unresolved groups its own Ẽ certifies the returned X̂ (certify()); OK when est·kCertSafety ≤ δ. An uncertified
// estimate that did not fall below kContract × the previous one — or fell so fast that the next sweep's quadratic
// part est³/est_prev² is below δ/8 while est ≤ 16δ (est_prev: the previous estimate, or ν = ‖X_k − X_{k−1}‖_F when
// the previous sweep had none) — sits at the truncation floor (quadratic in 2^-β,
// PAPER.md:341-373): θ grows by the power of 4 that brings it below δ/2, at most max_escalations times, then
// OZR_ERR_NOT_CONVERGED. Sweeps with unresolved groups (a Rayleigh–Ritz rotation, R13) are neither certified nor
// compared. Mirrors oracle/refine.refine_to_tol.
ozr_status ozr_refine_to_tol_dist(ozr_ctx ctx, ozr_comm comm, const double* A, int64_t n, int64_t lda, double* X,
                                  int64_t ldx, double* lambda, const ozr_params* params, ozr_step_report* history,
                                  int max_hist, int* sweeps_done) {
  ozr_status st = check_refine_args(ctx, comm, A, n, lda, X, ldx, lambda, params);
  if (st != OZR_OK) return st;
  SweepState ss;
  double est_prev = -1.0;
  int done = 0;
  ozr_status result = OZR_ERR_NOT_CONVERGED;
  ctx->err.clear();
  const int maxs = params->max_sweeps > 0 ? params->max_sweeps : 6;
  ozr_params P = effective_params(*params);
  int escalations = 0;
  Exchange* ex = comm ? comm->ex.get() : nullptr;
  const double delta = params->delta;
  for (int k = 0; k < maxs; ++k) {
    ozr_step_report rep;
    st = sweep(ctx, ex, A, n, lda, X, ldx, lambda, P, rep, ss);
    rep.theta = P.theta;
    rep.sweep = k + 1;
    rep.cert = -1.0;
    if (st == OZR_OK && rep.n_clusters == 0 && params->certify >= 1) st = certify(ctx, ex, n, delta, rep);
    if (st != OZR_OK) {
      if (sweeps_done) *sweeps_done = done;
      return st;
    }
    if (history && k < max_hist) history[k] = rep;
    done = k + 1;
    if (rep.n_clusters > 0 || params->certify < 1) {  // a Rayleigh–Ritz sweep: no certificate, no comparison
      est_prev = -1.0;
      continue;
    }
    const double est = rep.cert;
    if (est * kCertSafety <= delta) {
      result = OZR_OK;
      break;
    }
    // the first certified sweep after a start, a cluster sweep or an escalation has no previous estimate: there
    // ν = ‖X_k − X_{k−1}‖_F, the size of the error this sweep removed, stands in for it in the second test
    // (only while θ can still grow: without an escalation to spend, a floor read off ν would stop a run that the
    // next sweep may well finish — the untruncated and fixed-slice modes, or the escalations used up)
    const bool can_escalate = P.truncate && escalations < params->max_escalations;
    const double prev = est_prev > 0.0 ? est_prev : (can_escalate ? rep.net_update : -1.0);
    const bool floor = (est_prev > 0.0 && est > kContract * est_prev) ||
                       (prev > 0.0 && est <= 16.0 * delta && est * est * est / (prev * prev) <= delta / 8);
    if (floor) {
      if (P.truncate && escalations < params->max_escalations) {
        ++escalations;
        const int m = std::max(1, static_cast<int>(std::ceil(std::log(2.0 * est * kCertSafety / delta) / std::log(4.0))));
        P.theta = (P.theta > 0 ? P.theta : 1.0) * std::ldexp(1.0, 2 * std::min(m, 10));
        est_prev = -1.0;
        continue;
      }
      fail(ctx, OZR_ERR_NOT_CONVERGED, "stagnation at the truncation floor: certified error %.3e > delta %.3e", est,
           delta);
      break;
    }
    est_prev = est;
  }
  if (result != OZR_OK && ctx->err.empty()) fail(ctx, OZR_ERR_NOT_CONVERGED, "max_sweeps reached");
  if (sweeps_done) *sweeps_done = done;
  return guard_check(ctx, result);
}

ozr_status ozr_refine_step(ozr_ctx ctx, const double* A, int64_t n, int64_t lda, double* X, int64_t ldx,
                           double* lambda, const ozr_params* params, ozr_step_report* report) {
  return ozr_refine_step_dist(ctx, nullptr, A, n, lda, X, ldx, lambda, params, report);
}

ozr_status ozr_refine_to_tol(ozr_ctx ctx, const double* A, int64_t n, int64_t lda, double* X, int64_t ldx,
                             double* lambda, const ozr_params* params, ozr_step_report* history, int max_hist,
                             int* sweeps_done) {
  return ozr_refine_to_tol_dist(ctx, nullptr, A, n, lda, X, ldx, lambda, params, history, max_hist, sweeps_done);
}

}  // extern "C"
