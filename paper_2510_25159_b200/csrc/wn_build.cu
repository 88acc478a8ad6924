// wn_build.cu -- build side of libwn: segment prep (K1), lifting (K2a), the
// host planner that enumerates lattice copies / line terms / pairs (K2b, native
// C++), pairing probes run through the query kernel (Algs. 7-9), and record
// emission (K2c).  PAPER.md is cited as P:<line>.
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <omp.h>
#include <numeric>
#include <vector>

#include "wn_common.cuh"

namespace wn {

static thread_local char g_err[512] = "";

// WN_TRACE=1: host-side phase timings of wn_build_faces on stderr, with stream
// synchronisations after the kernel groups (device phase times); WN_TRACE=2:
// host timestamps only (no added synchronisation)
struct Trace {
  bool on = std::getenv("WN_TRACE") != nullptr;
  bool sync = on && std::atoi(std::getenv("WN_TRACE")) == 1;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now(), last = t0;
  void mark(const char *what) {
    if (!on) return;
    auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[wn_build] %-28s %8.3f ms (total %8.3f)\n", what,
            std::chrono::duration<double, std::milli>(now - last).count(),
            std::chrono::duration<double, std::milli>(now - t0).count());
    last = now;
  }
};
thread_local int32_t g_build_launches = 0;

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

wn_status_t cuda_fail(cudaError_t e, const char *what) {
  set_error("CUDA error %s (%s) in %s", cudaGetErrorName(e), cudaGetErrorString(e), what);
  return (e == cudaErrorMemoryAllocation) ? WN_ERR_NOMEM : WN_ERR_CUDA;
}

// ---------------------------------------------------------------------------
// K0: degree check -> control-point counts (prefix-summed into offsets)
// ---------------------------------------------------------------------------
__global__ void k_deg(int32_t n_segs, const int32_t *__restrict__ deg, int32_t *__restrict__ cnt,
                      int32_t *__restrict__ bad) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s > n_segs) return;
  if (s == n_segs) { cnt[s] = 0; return; }
  const int n = deg[s];
  const bool ok = n >= 1 && n <= 5;
  cnt[s] = ok ? n + 1 : 0;
  if (!ok) atomicOr(bad, 1);
}

// ---------------------------------------------------------------------------
// K1: segment prep.  Derivative bound B of Lemma 1: polynomial
// hodograph bound max_i n|P_i - P_{i-1}|; rational: Floater's
// two bounds n(W/w)max|P_i-P_j| and n(W/w)^2 max|P_i-P_{i-1}| (P:1101-1109,
// reading R8), and the Bernstein bound of the hodograph numerator
// max_k |D_k| / min_k E_k (reading R29; D = X'W - XW' of degree 2n-1, E = W^2
// of degree 2n in Bernstein form).  B = the minimum of the valid bounds.  Root
// span S0 = min(B, control-polygon length) (R9).  Piece bounds Bq[8]: the same
// bound on the 8 dyadic pieces [q/8,(q+1)/8] (homogeneous de Casteljau, t-units),
// used for sub-spans inside one piece (Eq. 2 with the piece's own bound).
// ---------------------------------------------------------------------------
// Exact binomial coefficients, constant-folded in the unrolled bound code.
__host__ __device__ constexpr double binom_c(int n, int k) {
  double r = 1.0;
  for (int i = 1; i <= k; ++i) r = r * (n - k + i) / i;
  return r;
}

// Bounds on homogeneous control points (X_i, Y_i, W_i) = w_i (x_i, y_i, 1),
// i = 0..N, held in registers (templated on the degree, fully unrolled).
// Written without accumulating into local arrays (an earlier version of that
// shape was miscompiled by nvcc 12.9 -O3 on sm_100a: scripts/dev/kp.cu).
// Norms are compared squared and rooted once; the bounds' rounding (a few
// ulps) is covered by the (1 + 2^-40) factor k_emit applies (R5).
//
// Hodograph-numerator Bernstein bound: |gamma'| = |X'W - XW'| / W^2 with
//   X'W - XW' = N sum_k D_k B_k^{2N-1},
//   D_k = sum_{i+j=k} C(N-1,i)C(N,j)/C(2N-1,k) [W_j (X_{i+1}-X_i) - (W_{i+1}-W_i) X_j],
//   W^2 = sum_k E_k B_k^{2N},  E_k = sum_{i+j=k} C(N,i)C(N,j)/C(2N,k) W_i W_j,
// so |gamma'| <= N max_k |D_k| / min_k E_k (convex-hull property).
template <int N>
__device__ __forceinline__ double hodo_bound(const double (&X)[N + 1], const double (&Y)[N + 1],
                                             const double (&W)[N + 1]) {
  double d2max = 0.0, emin = INFINITY;
#pragma unroll
  for (int k = 0; k <= 2 * N - 1; ++k) {
    double dx = 0.0, dy = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const int j = k - i;
      if (j < 0 || j > N) continue;
      const double c = binom_c(N - 1, i) * binom_c(N, j) / binom_c(2 * N - 1, k);
      dx += c * (W[j] * (X[i + 1] - X[i]) - (W[i + 1] - W[i]) * X[j]);
      dy += c * (W[j] * (Y[i + 1] - Y[i]) - (W[i + 1] - W[i]) * Y[j]);
    }
    d2max = fmax(d2max, dx * dx + dy * dy);
  }
#pragma unroll
  for (int k = 0; k <= 2 * N; ++k) {
    double e = 0.0;
#pragma unroll
    for (int i = 0; i <= N; ++i) {
      const int j = k - i;
      if (j < 0 || j > N) continue;
      e += (binom_c(N, i) * binom_c(N, j) / binom_c(2 * N, k)) * W[i] * W[j];
    }
    emin = fmin(emin, e);
  }
  return N * sqrt(d2max) / emin;
}

// Floater's rational bounds on the affine control points (x_i, y_i) and weights
template <int N>
__device__ __forceinline__ double floater_bound(const double (&px)[N + 1], const double (&py)[N + 1],
                                                const double (&W)[N + 1]) {
  double wmax = W[0], wmin = W[0], d2max = 0.0, diam2 = 0.0;
#pragma unroll
  for (int i = 1; i <= N; ++i) { wmax = fmax(wmax, W[i]); wmin = fmin(wmin, W[i]); }
#pragma unroll
  for (int i = 0; i <= N; ++i)
#pragma unroll
    for (int j = i + 1; j <= N; ++j) {
      const double dx = px[j] - px[i], dy = py[j] - py[i];
      const double l2 = dx * dx + dy * dy;
      diam2 = fmax(diam2, l2);
      if (j == i + 1) d2max = fmax(d2max, l2);
    }
  const double dmax = sqrt(d2max);
  if (wmax == wmin) return N * dmax;
  const double r = wmax / wmin;
  return fmin(N * r * sqrt(diam2), N * r * r * dmax);
}

// Subdivision matrices of the dyadic pieces [q/8, (q+1)/8]: piece control
// point i = sum_j S[N][q][i][j] P_j.  Generated at compile time by three de
// Casteljau halvings of the unit control vectors (entries are dyadic
// rationals with denominators <= 2^15: exact in double).
struct SubTab {
  double m[5][8][6][6];
};
constexpr SubTab make_subtab() {
  SubTab T{};
  for (int N = 1; N <= 5; ++N)
    for (int q = 0; q < 8; ++q)
      for (int col = 0; col <= N; ++col) {
        double a[6] = {0, 0, 0, 0, 0, 0};
        a[col] = 1.0;
        for (int lvl = 2; lvl >= 0; --lvl) {
          const bool right = (q >> lvl) & 1;
          double t[6] = {a[0], a[1], a[2], a[3], a[4], a[5]};
          double o[6] = {0, 0, 0, 0, 0, 0};
          o[0] = t[0];
          o[N] = t[N];
          // after round r, entry 0 is the left half's point r, entry N-r the right half's
          for (int r = 1; r <= N; ++r) {
            for (int j = 0; j <= N - r; ++j) t[j] = 0.5 * (t[j] + t[j + 1]);
            if (right) o[N - r] = t[N - r];
            else o[r] = t[0];
          }
          if (right) o[N] = a[N];
          else o[0] = a[0];
          for (int i = 0; i <= N; ++i) a[i] = o[i];
        }
        for (int i = 0; i <= N; ++i) T.m[N - 1][q][i][col] = a[i];
      }
  return T;
}
__constant__ SubTab c_sub = make_subtab();
#ifndef PREP_MINB
#define PREP_MINB 4
#endif

template <int N>
__device__ __forceinline__ void dyadic_piece(const double (&X)[N + 1], const double (&Y)[N + 1],
                                             const double (&W)[N + 1], int q, double (&a)[N + 1],
                                             double (&b)[N + 1], double (&c)[N + 1]) {
#pragma unroll
  for (int i = 0; i <= N; ++i) {
    double sa = 0.0, sb = 0.0, sc = 0.0;
#pragma unroll
    for (int j = 0; j <= N; ++j) {
      const double m = c_sub.m[N - 1][q][i][j];
      sa = fma(m, X[j], sa);
      sb = fma(m, Y[j], sb);
      sc = fma(m, W[j], sc);
    }
    a[i] = sa; b[i] = sb; c[i] = sc;
  }
}

// Control-polygon length of a (homogeneous) piece: an upper bound on its arc
// length (rational de Casteljau cuts corners of the projected polygon).
template <int N>
__device__ __forceinline__ double poly_len(const double (&a)[N + 1], const double (&b)[N + 1],
                                           const double (&c)[N + 1]) {
  // (plain sqrt: coordinates are far from overflow; rounding ~1e-16 relative is
  // covered by the R5 margins like every other bound)
  double r = 1.0 / c[0];
  double L = 0.0, x0 = a[0] * r, y0 = b[0] * r;
#pragma unroll
  for (int i = 1; i <= N; ++i) {
    r = 1.0 / c[i];
    const double x1 = a[i] * r, y1 = b[i] * r;
    L += sqrt((x1 - x0) * (x1 - x0) + (y1 - y0) * (y1 - y0));
    x0 = x1;
    y0 = y1;
  }
  return L;
}

// K1 output sinks.  PrepSink: the diagnostics record of wn_segment_prep
// (unmargined doubles).  ColdSink<R>: the build's base cold record of the
// segment (margins applied, piece bounds rounded up to fp32: still upper
// bounds) plus its root span S0 (unmargined) for the hierarchy prefix sums and
// the hot SEG record.  Both are fed by the same bound code (prep_n).
struct PrepSink {
  static constexpr bool kStaged = false;
  using Rec = SegPrep;
  SegPrep *out;
  __device__ void at(int, int, SegPrep *) {}
  __device__ void zero(int s) const {
    double2 *o2 = reinterpret_cast<double2 *>(out + s);
    for (int k = 0; k < 9; ++k) o2[k] = make_double2(0.0, 0.0);
  }
  __device__ void pieces(int s, int q, double B, double b0, double b1, double l0, double l1) const {
    double2 *o2 = reinterpret_cast<double2 *>(out + s);
    o2[1 + q / 2] = make_double2(b0, b1);
    o2[5 + q / 2] = make_double2(l0, l1);
  }
  template <int N>
  __device__ void head(int, double, const double *, const double *, const double *) const {}
  __device__ void tail(int s, double B, double S0) const { reinterpret_cast<double2 *>(out + s)[0] = make_double2(B, S0); }
};

__device__ __forceinline__ float f_dn(double x) { return __double2float_rd(x); }
__device__ __forceinline__ float f_up(double x) { return __double2float_ru(x); }

// C(n, j) for 0 <= j <= n <= 5, exact: 4-bit entries of a packed table indexed
// by 6 n + j (no divisions, no local or constant-memory table)
__device__ __forceinline__ double binom5(int n, int j) {
  constexpr unsigned long long T0 = 0x0000000000000000ull   // n = 0, 1, 2 (idx 0..15)
      | 1ull << 0                                            // C(0,0)
      | 1ull << 24 | 1ull << 28                              // C(1,0..1)
      | 1ull << 48 | 2ull << 52 | 1ull << 56;                // C(2,0..2)
  constexpr unsigned long long T1 = 0x0000000000000000ull   // n = 3, 4, 5 (idx 18..35, minus 18)
      | 1ull << 0 | 3ull << 4 | 3ull << 8 | 1ull << 12        // C(3,0..3)
      | 1ull << 24 | 4ull << 28 | 6ull << 32 | 4ull << 36 | 1ull << 40   // C(4,0..4)
      | 1ull << 48 | 5ull << 52 | 10ull << 56 | 10ull << 60;           // C(5,0..3)
  const int idx = 6 * n + j;
  unsigned v;
  if (idx < 18) v = (unsigned)(T0 >> (4 * idx)) & 15u;
  else if (idx < 34) v = (unsigned)(T1 >> (4 * (idx - 18))) & 15u;
  else v = idx == 34 ? 5u : 1u;                              // C(5,4), C(5,5)
  return (double)v;
}

template <typename R>
struct ColdSink {
  // The records are indexed by the segment's position p in the degree-sorted
  // order (inv[s] = p): a K1 CTA's records are then contiguous, assembled in
  // shared memory (slot) and written with one bulk copy (coalesced).
  static constexpr bool kStaged = true;
  using Rec = BaseCold<R>;
  BaseCold<R> *out;    // [p]
  double *s0;          // [s] root span S0
  int32_t *inv;        // [s] -> p
  double rel;          // relative margin (R5): 2^-40 fp64, 2^-17 fp32
  BaseCold<R> *slot;   // record under assembly (shared memory; global for k_prep_bad)
  __device__ void at(int p, int s, BaseCold<R> *where) {
    slot = where;
    inv[s] = p;
  }
  __device__ void zero(int s) const {
    uint4 *o = reinterpret_cast<uint4 *>(slot);
    for (int k = 0; k < (int)(sizeof(BaseCold<R>) / 16); ++k) o[k] = make_uint4(0, 0, 0, 0);
    s0[s] = 0.0;
  }
  // Piece bounds go to Bq.  The spans of the depth-1..3 nodes are built as the
  // pieces arrive (q = 0, 2, 4, 6 with their right neighbours): depth 3 = the
  // piece itself, depth 2 = the pair, depth 1 = two pairs (running max / sum in
  // scalars); min(2^-d max Bq, sum Lq) from the margined doubles, rounded up.
  double acc_b = 0.0, acc_l = 0.0;
  __device__ void pieces(int, int q, double B, double b0, double b1, double l0, double l1) {
    BaseCold<R> *C = slot;
    const double m0 = fmin(B, b0) * (1.0 + rel), m1 = fmin(B, b1) * (1.0 + rel);
    const double L0 = l0 * (1.0 + rel), L1 = l1 * (1.0 + rel);
    *reinterpret_cast<float2 *>(&C->Bq[q]) = make_float2(f_up(m0), f_up(m1));
    // depth 3 (index 6 + q), depth 2 (index 2 + q/2)
    *reinterpret_cast<float2 *>(&C->Sp[6 + q]) = make_float2(f_up(fmin(ldexp(m0, -3), L0)), f_up(fmin(ldexp(m1, -3), L1)));
    const double pb = fmax(m0, m1), pl = L0 + L1;
    C->Sp[2 + q / 2] = f_up(fmin(ldexp(pb, -2), pl));
    if ((q & 2) == 0) {
      acc_b = pb;
      acc_l = pl;
    } else {                                               // depth 1 (index q / 4)
      C->Sp[q / 4] = f_up(fmin(ldexp(fmax(acc_b, pb), -1), acc_l + pl));
    }
  }
  // end points (exact, stored coordinates), bound, degree, homogeneous Horner
  // coefficients c_j = (C(n,j) w_j) (x_j, y_j, 1), zero above the degree
  __device__ void tail(int s, double, double S0) const { s0[s] = S0; }
  // written before the piece loop so that the control points die early
  template <int N>
  __device__ void head(int, double B, const double *px, const double *py, const double *W) const {
    BaseCold<R> *C = slot;
    *reinterpret_cast<double2 *>(&C->x0) = make_double2(px[0], py[0]);
    *reinterpret_cast<double2 *>(&C->xn) = make_double2(px[N], py[N]);
    const double Bm = B * (1.0 + rel);
    if constexpr (sizeof(R) == 8) {
      *reinterpret_cast<double2 *>(&C->B) = make_double2(Bm, __longlong_as_double((long long)N));
#pragma unroll
      for (int j = 0; j < 6; j += 2) {
        double cx2[2], cy2[2], cw2[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int jj = j + h;
          cx2[h] = cy2[h] = cw2[h] = 0.0;
          if (jj <= N) {
            const double cw = binom5(N, jj) * W[jj];
            cx2[h] = cw * px[jj];
            cy2[h] = cw * py[jj];
            cw2[h] = cw;
          }
        }
        *reinterpret_cast<double2 *>(&C->cx[j]) = make_double2(cx2[0], cx2[1]);
        *reinterpret_cast<double2 *>(&C->cy[j]) = make_double2(cy2[0], cy2[1]);
        *reinterpret_cast<double2 *>(&C->cw[j]) = make_double2(cw2[0], cw2[1]);
      }
    } else {
      C->B = f_up(Bm);
      C->n = N;
#pragma unroll
      for (int jj = 0; jj < 6; ++jj) {
        float cx = 0.f, cy = 0.f, cwf = 0.f;
        if (jj <= N) {
          const double cw = binom5(N, jj) * W[jj];
          cx = (float)(cw * px[jj]);
          cy = (float)(cw * py[jj]);
          cwf = (float)cw;
        }
        C->cx[jj] = cx;
        C->cy[jj] = cy;
        C->cw[jj] = cwf;
      }
    }
  }
};

// One thread per segment (taken in degree-sorted order so that a warp runs one
// degree variant): loads its control points once and computes B, S0 and the 8
// piece bounds and piece polygon lengths, written through the sink.
template <int N, class Sink>
__device__ __forceinline__ void prep_n(const double *__restrict__ ctrl, const double *__restrict__ w, int o, int s,
                                       Sink &sink, uint8_t *__restrict__ err_out) {
  double X[N + 1], Y[N + 1], W[N + 1], px[N + 1], py[N + 1];
  bool err = false;
  double lpoly = 0.0;
#pragma unroll
  for (int j = 0; j <= N; ++j) {
    const double x = ctrl[2 * (o + j)], y = ctrl[2 * (o + j) + 1], wj = w ? w[o + j] : 1.0;
    err |= !isfinite(x) || !isfinite(y) || !isfinite(wj) || !(wj > 0.0);
    X[j] = wj * x; Y[j] = wj * y; W[j] = wj;
    px[j] = x; py[j] = y;
    if (j) lpoly += hypot(x - px[j - 1], y - py[j - 1]);
  }
  err_out[s] = err ? 1 : 0;
  if (err) {
    sink.zero(s);
    return;
  }
  const double B = fmin(floater_bound<N>(px, py, W), hodo_bound<N>(X, Y, W));
  sink.template head<N>(s, B, px, py, W);
  double l8 = 0.0;   // sum of the 8 dyadic pieces' polygon lengths >= arc length (R9, tighter)
#pragma unroll 1
  for (int q = 0; q < 8; q += 2) {
    double a[N + 1], bb[N + 1], c[N + 1];
    dyadic_piece<N>(X, Y, W, q, a, bb, c);
    const double b0 = 8.0 * hodo_bound<N>(a, bb, c);
    const double l0 = poly_len<N>(a, bb, c);
    dyadic_piece<N>(X, Y, W, q + 1, a, bb, c);
    const double b1 = 8.0 * hodo_bound<N>(a, bb, c);
    const double l1 = poly_len<N>(a, bb, c);
    l8 += l0 + l1;
    sink.pieces(s, q, B, b0, b1, l0, l1);
  }
  sink.tail(s, B, fmin(B, fmin(lpoly, l8)));
}

#ifndef PREP_SPLIT
#define PREP_SPLIT 8   // CTAs per SM of the per-degree K1 kernels
#endif
#ifndef K1_STREAMS
#define K1_STREAMS 1   // 1: the per-degree K1 kernels run concurrently on side streams
#endif
// Per-degree K1: the degree-sorted segments split into the ranges of the sort
// key (deg & 7, the radix sort's 3 bits) so that each degree variant runs with
// its own register budget (degree 1-3 need far fewer than degree 5).  bnd[k] =
// first sorted position with key >= k, k = 0..8.
__global__ void k_deg_bounds(int32_t n, const int32_t *__restrict__ sdeg, int32_t *__restrict__ bnd) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p > n) return;
  const int prev = p ? (sdeg[p - 1] & 7) : -1;
  const int cur = p < n ? (sdeg[p] & 7) : 8;
  for (int k = prev + 1; k <= cur; ++k) bnd[k] = p;
}

#ifndef PREP_DEG_MINB
#define PREP_DEG_MINB 4   // 128 registers: degree 5 spills 72 B but runs at 4 CTAs / SM (measured faster than 1-3)
#endif
template <int N, class Sink>
__global__ void __launch_bounds__(128, PREP_DEG_MINB) k_prep_deg(const int32_t *__restrict__ bnd, const int32_t *__restrict__ deg,
                                                  const int32_t *__restrict__ coff, const double *__restrict__ ctrl,
                                                  const double *__restrict__ w, Sink sink,
                                                  uint8_t *__restrict__ serr, const int32_t *__restrict__ order) {
  const int lo = bnd[N], hi = bnd[N + 1];
  if constexpr (Sink::kStaged) {
    // records of this CTA's 128 consecutive sorted positions assembled in
    // shared memory, then written out with one 1-D bulk copy (TMA store)
    extern __shared__ __align__(128) unsigned char k1_stage[];
    using Rec = typename Sink::Rec;
    Rec *stage = reinterpret_cast<Rec *>(k1_stage);
    for (int base = lo + blockIdx.x * blockDim.x; base < hi; base += gridDim.x * blockDim.x) {
      const int p = base + threadIdx.x;
      WN_DCHECK(blockDim.x <= 128);
      if (p < hi) {
        const int s = order[p];
        sink.at(p, s, stage + threadIdx.x);
        if (deg[s] == N) {
          prep_n<N>(ctrl, w, coff[s], s, sink, serr);
        } else {   // a degree outside 1..5 with these low bits (rejected on the host)
          serr[s] = 1;
          sink.zero(s);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> async proxy
      __syncthreads();
      if (threadIdx.x == 0) {
        const unsigned bytes = (unsigned)(min((int)blockDim.x, hi - base) * sizeof(Rec));
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(sink.out + base),
                     "r"((unsigned)__cvta_generic_to_shared(stage)), "r"(bytes)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");   // stage reusable
      }
      __syncthreads();
    }
  } else {
    for (int p = lo + blockIdx.x * blockDim.x + threadIdx.x; p < hi; p += gridDim.x * blockDim.x) {
      const int s = order[p];
      if (deg[s] == N) {
        prep_n<N>(ctrl, w, coff[s], s, sink, serr);
      } else {   // a degree outside 1..5 with these low bits (rejected on the host)
        serr[s] = 1;
        sink.zero(s);
      }
    }
  }
}

// keys 0, 6, 7: degrees outside 1..5 only
template <class Sink>
__global__ void k_prep_bad(const int32_t *__restrict__ bnd, Sink sink, uint8_t *__restrict__ serr,
                           const int32_t *__restrict__ order) {
  const int n0 = bnd[1] - bnd[0], n1 = bnd[8] - bnd[6];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n0 + n1; i += gridDim.x * blockDim.x) {
    const int p = i < n0 ? bnd[0] + i : bnd[6] + (i - n0);
    const int s = order[p];
    serr[s] = 1;
    if constexpr (Sink::kStaged) sink.at(p, s, sink.out + p);
    sink.zero(s);
  }
}

__global__ void k_iota(int32_t n, int32_t *__restrict__ a) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = i;
}

__global__ void k_loop_face(int32_t n_faces, int32_t n_loops, const int32_t *__restrict__ face_off,
                            int32_t *__restrict__ loop_face) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= n_faces) return;
  const int l0 = max(face_off[f], 0), l1 = min(face_off[f + 1], n_loops);   // clamped (validated on the host)
  for (int l = l0; l < l1; ++l) loop_face[l] = f;
}


// ---------------------------------------------------------------------------
// K2a: lifting to the universal covering space (Sec. 4.3).  Loops
// are stored seam-discontinuously (R18); segment i is translated by the lattice
// vector nearest to continuing from the lifted end of segment i-1 (R17/R18).
// Homology class = round(closure / T).  Junctions that are not
// bit-continuous after lifting are recorded as chain breaks.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256, 4) k_lift(int32_t n_loops, int32_t n_faces, int32_t n_segs,
                                              const int32_t *__restrict__ loop_off,
                                              const int32_t *__restrict__ loop_face,
                                              const uint8_t *__restrict__ face_per, const double *__restrict__ face_dom,
                                              const int32_t *__restrict__ deg, const int32_t *__restrict__ coff,
                                              const double *__restrict__ ctrl, const double *__restrict__ wts,
                                              int2 *__restrict__ shift, uint8_t *__restrict__ brk,
                                              int2 *__restrict__ chain, double2 *__restrict__ lsta,
                                              double2 *__restrict__ lend,
                                              LoopInfo *__restrict__ info) {
  // one warp per loop; lanes take its segments 32 at a time.  The lattice
  // shifts are a sequential recurrence (each segment continues from the
  // lifted end of the previous one, R17/R18): the warp walks a chunk's 32
  // segments in order with broadcast end points; everything else is parallel.
  const int l = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (l >= n_loops) return;
  const int f = loop_face[l];
  const bool fok = f >= 0 && f < n_faces;   // -1: loop outside every face (bad CSR, rejected on the host)
  const int pu = fok ? face_per[f] & 1 : 0, pv = fok ? (face_per[f] >> 1) & 1 : 0;
  const double Tu = fok ? face_dom[4 * f + 1] : 0.0, Tv = fok ? face_dom[4 * f + 3] : 0.0;
  const int s0 = min(max(loop_off[l], 0), n_segs), s1 = min(max(loop_off[l + 1], s0), n_segs);
  double ex = 0, ey = 0;           // lifted end of the previous segment (uniform)
  double sx = 0, sy = 0;
  int nbrk = 0, err = 0, cs = 0;   // cs: chain start (loop index) carried across chunks
  int cku = 0, ckv = 0;            // shift of the previous chunk's last segment
  double cxr = 0, cyr = 0;         // its raw (stored) end point
  double xmin = INFINITY, ymin = INFINITY, xmax = -INFINITY, ymax = -INFINITY;
  for (int base = s0; base < s1; base += 32) {
    const int s = base + lane;
    const bool in = s < s1;
    const int cnt = min(32, s1 - base);
    double x0 = 0, y0 = 0, xe = 0, ye = 0, bx0 = INFINITY, by0 = INFINITY, bx1 = -INFINITY, by1 = -INFINITY;
    bool e = false;
    if (in) {
      int n = deg[s];
      const int o = coff[s];
      if (n < 1 || n > 5) { e = true; n = -1; }   // rejected on the host (k_deg flag)
      for (int j = 0; j <= n; ++j) {
        const double x = ctrl[2 * (o + j)], y = ctrl[2 * (o + j) + 1], wj = wts ? wts[o + j] : 1.0;
        e |= !isfinite(x) || !isfinite(y) || !isfinite(wj) || !(wj > 0.0);
        bx0 = fmin(bx0, x); bx1 = fmax(bx1, x);
        by0 = fmin(by0, y); by1 = fmax(by1, y);
        if (j == 0) { x0 = x; y0 = y; }
        if (j == n) { xe = x; ye = y; }
      }
    }
    err |= __any_sync(0xffffffffu, e);
    // shifts (R17/R18): k_s = round((lifted end of s-1 - start of s) / T),
    // k = 0 for the loop's first segment -- a sequential recurrence.  The
    // candidates are the prefix sums of the local deltas round((raw end of s-1
    // - start of s) / T); every lane then re-evaluates the recurrence with its
    // candidate predecessor, so if all agree the candidates ARE the recurrence's
    // values (induction from k = 0).  A chunk where a lane disagrees (a rounding
    // tie) walks the recurrence serially.
    int ku = 0, kv = 0;
    if (pu || pv) {
      const bool first = s == s0;
      double pxr = __shfl_up_sync(0xffffffffu, xe, 1), pyr = __shfl_up_sync(0xffffffffu, ye, 1);
      if (lane == 0) { pxr = cxr; pyr = cyr; }
      int su = 0, sv = 0;
      if (in && !first) {
        if (pu) su = (int)round(__ddiv_rn(__dsub_rn(pxr, x0), Tu));
        if (pv) sv = (int)round(__ddiv_rn(__dsub_rn(pyr, y0), Tv));
      }
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int tu = __shfl_up_sync(0xffffffffu, su, o), tv = __shfl_up_sync(0xffffffffu, sv, o);
        if (lane >= o) { su += tu; sv += tv; }
      }
      ku = cku + su;
      kv = ckv + sv;
      int pku = __shfl_up_sync(0xffffffffu, ku, 1), pkv = __shfl_up_sync(0xffffffffu, kv, 1);
      if (lane == 0) { pku = cku; pkv = ckv; }
      bool ok = true;
      if (in && !first) {
        if (pu) ok &= ku == (int)round(__ddiv_rn(__dsub_rn(lat(pxr, pku, Tu), x0), Tu));
        if (pv) ok &= kv == (int)round(__ddiv_rn(__dsub_rn(lat(pyr, pkv, Tv), y0), Tv));
      }
      if (!__all_sync(0xffffffffu, ok)) {
        double qx = ex, qy = ey;   // lifted end of the previous segment
        for (int j = 0; j < cnt; ++j) {
          const double x0j = __shfl_sync(0xffffffffu, x0, j), y0j = __shfl_sync(0xffffffffu, y0, j);
          const double xej = __shfl_sync(0xffffffffu, xe, j), yej = __shfl_sync(0xffffffffu, ye, j);
          int kuj = 0, kvj = 0;
          if (base + j > s0) {
            if (pu) kuj = (int)round(__ddiv_rn(__dsub_rn(qx, x0j), Tu));
            if (pv) kvj = (int)round(__ddiv_rn(__dsub_rn(qy, y0j), Tv));
          }
          if (lane == j) { ku = kuj; kv = kvj; }
          qx = pu ? lat(xej, kuj, Tu) : xej;
          qy = pv ? lat(yej, kvj, Tv) : yej;
        }
      }
    }
    // lifted start / end, the previous lifted end, bit-continuity of the junction
    const double lx0 = pu ? lat(x0, ku, Tu) : x0, ly0 = pv ? lat(y0, kv, Tv) : y0;
    const double lxe = pu ? lat(xe, ku, Tu) : xe, lye = pv ? lat(ye, kv, Tv) : ye;
    double pex = __shfl_up_sync(0xffffffffu, lxe, 1), pey = __shfl_up_sync(0xffffffffu, lye, 1);
    if (lane == 0) { pex = ex; pey = ey; }
    const bool bk = in && s > s0 && !(lx0 == pex && ly0 == pey);
    if (base == s0) { sx = __shfl_sync(0xffffffffu, lx0, 0); sy = __shfl_sync(0xffffffffu, ly0, 0); }
    ex = __shfl_sync(0xffffffffu, lxe, cnt - 1);
    ey = __shfl_sync(0xffffffffu, lye, cnt - 1);
    cku = __shfl_sync(0xffffffffu, ku, cnt - 1);
    ckv = __shfl_sync(0xffffffffu, kv, cnt - 1);
    cxr = __shfl_sync(0xffffffffu, xe, cnt - 1);
    cyr = __shfl_sync(0xffffffffu, ye, cnt - 1);
    if (in) {
      shift[s] = make_int2(ku, kv);
      brk[s] = bk;
      lsta[s] = make_double2(lx0, ly0);     // lifted start / end: the emission's chain points
      // lifted box and end point: lat() is monotone, so it commutes with min/max
      bx0 = pu ? lat(bx0, ku, Tu) : bx0; bx1 = pu ? lat(bx1, ku, Tu) : bx1;
      by0 = pv ? lat(by0, kv, Tv) : by0; by1 = pv ? lat(by1, kv, Tv) : by1;
      lend[s] = make_double2(lxe, lye);
    }
    xmin = fmin(xmin, bx0); xmax = fmax(xmax, bx1);
    ymin = fmin(ymin, by0); ymax = fmax(ymax, by1);
    // chain starts: the last break (or the loop start) at or before s
    const unsigned bm = __ballot_sync(0xffffffffu, in && (bk || s == s0));
    nbrk += __popc(__ballot_sync(0xffffffffu, in && bk));
    const unsigned upto = bm & ((2u << lane) - 1u);
    const int my_cs = upto ? (base + 31 - __clz(upto)) - s0 : cs;
    if (in) chain[s].x = my_cs;
    if (bm) cs = (base + 31 - __clz(bm)) - s0;
  }
  // chain lengths: next chain start after s (backward over the chunks)
  __syncwarp();
  int nxt = s1 - s0;                 // first chain start after the current chunk
  for (int base = s0 + ((s1 - s0 - 1) / 32) * 32; base >= s0 && s1 > s0; base -= 32) {
    const int s = base + lane;
    const bool in = s < s1;
    const bool st = in && (s == s0 || brk[s]);
    const unsigned bm = __ballot_sync(0xffffffffu, st);
    const unsigned after = bm & ~((2u << lane) - 1u);   // chain starts strictly after s
    const int ce = after ? (base + __ffs(after) - 1) - s0 : nxt;
    if (in) chain[s].y = ce - chain[s].x;
    if (bm) nxt = (base + __ffs(bm) - 1) - s0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    xmin = fmin(xmin, __shfl_xor_sync(0xffffffffu, xmin, o));
    ymin = fmin(ymin, __shfl_xor_sync(0xffffffffu, ymin, o));
    xmax = fmax(xmax, __shfl_xor_sync(0xffffffffu, xmax, o));
    ymax = fmax(ymax, __shfl_xor_sync(0xffffffffu, ymax, o));
  }
  if (lane == 0) {
    LoopInfo I;
    I.cu = (pu && s1 > s0) ? (int)round(__ddiv_rn(__dsub_rn(ex, sx), Tu)) : 0;
    I.cv = (pv && s1 > s0) ? (int)round(__ddiv_rn(__dsub_rn(ey, sy), Tv)) : 0;
    I.nbrk = nbrk;
    I.closed = (s1 > s0) && ex == sx && ey == sy;
    I.err = err;
    I.nseg = s1 - s0;
    I.sx = sx;
    I.sy = sy;
    I.bb[0] = xmin; I.bb[1] = ymin; I.bb[2] = xmax; I.bb[3] = ymax;
    info[l] = I;
  }
}

// prefix sums of the root spans S0 along each loop (warp per loop, after K1);
// the path-hierarchy spans are differences of them.  Summation
// order differs from a serial sum by a few ulps, far inside the R5 margin.
__global__ void __launch_bounds__(256) k_s0pre(int32_t n_loops, int32_t n_segs, const int32_t *__restrict__ loop_off,
                                               const double *__restrict__ seg_s0, double *__restrict__ s0pre) {
  const int l = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (l >= n_loops) return;
  const int s0 = min(max(loop_off[l], 0), n_segs), s1 = min(max(loop_off[l + 1], s0), n_segs);
  double carry = 0.0;
  for (int base = s0; base < s1; base += 32) {
    const int s = base + lane;
    double v = s < s1 ? seg_s0[s] : 0.0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double u = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += u;
    }
    v += carry;
    if (s < s1) s0pre[s] = v;
    carry = __shfl_sync(0xffffffffu, v, 31);
  }
}

// ---------------------------------------------------------------------------
// K2c: record emission, one thread per planned group.
// ---------------------------------------------------------------------------
// Path-hierarchy trees of closed single-chain loops omit their top OMIT_LEVELS
// levels of SPAN nodes: the half-loop ellipses of a closed loop contain
// (nearly) the whole loop interior, so those nodes almost never prune and a
// warp would only spend an iteration descending them.  Value-neutral (an
// omitted node = always descend).  Split rule of every tree: [a, b] ->
// [a, mid], [mid + 1, b], mid = (a + b) >> 1.
constexpr int OMIT_LEVELS = 2;
static_assert(OMIT_LEVELS <= 2, "tree_internal_top is written out for k <= 2");
__host__ __device__ inline int tree_internal_top(int n, int k) {   // internal nodes at depth < k
  int c = 0;
  if (k >= 1 && n >= 2) {
    ++c;
    if (k >= 2) {
      const int left = (n + 1) >> 1, right = n - left;   // left = mid - a + 1 for any [a, b]
      c += (left >= 2 ? 1 : 0) + (right >= 2 ? 1 : 0);
    }
  }
  return c;
}
// records of the pre-order tree over n leaves with its top k levels omitted
__host__ __device__ inline int tree_recs(int n, int k) { return 2 * n - 1 - tree_internal_top(n, k); }

template <typename R>
struct Emit;

// write a point-like record: (x, y) exact, s = span of the conservative filter
template <typename R>
__device__ void put_rec(Hot<R> *H, int r, double x, double y, double s, uint32_t meta);
template <>
__device__ void put_rec<double>(Hot<double> *H, int r, double x, double y, double s, uint32_t meta) {
  Hot<double> h;
  h.fx = __double2float_rn(x);
  h.fy = __double2float_rn(y);
  h.fs = f_up(s);
  h.meta = meta;
  h.x = x;
  h.y = y;
  H[r] = h;
}
template <>
__device__ void put_rec<float>(Hot<float> *H, int r, double x, double y, double s, uint32_t meta) {
  Hot<float> h;
  h.a = __double2float_rn(x);
  h.b = __double2float_rn(y);
  h.c = f_up(s);
  h.meta = meta;
  H[r] = h;
}

template <typename R>
__device__ void put_group(Hot<R> *H, int r, double xmin, double ymin, double xmax, double ymax, uint32_t meta);
template <>
__device__ void put_group<double>(Hot<double> *H, int r, double xmin, double ymin, double xmax, double ymax,
                                  uint32_t meta) {
  Hot<double> h;
  h.fx = f_dn(xmin);
  h.fy = f_dn(ymin);
  h.fs = f_up(xmax);
  h.meta = meta;
  h.x = __hiloint2double(0, __float_as_int(f_up(ymax)));   // fp32 ymax (rounded up) in the low word
  h.y = 0.0;
  H[r] = h;
}
template <>
__device__ void put_group<float>(Hot<float> *H, int r, double xmin, double ymin, double xmax, double ymax,
                                 uint32_t meta) {
  Hot<float> h;
  h.a = f_dn(xmin);
  h.b = f_dn(ymin);
  __half2 hi = __halves2half2(__float2half_ru(f_up(xmax)), __float2half_ru(f_up(ymax)));
  memcpy(&h.c, &hi, 4);
  h.meta = meta;
  H[r] = h;
}

// one warp per planned group; lanes take the group's segments in parallel.
// The path-hierarchy SPAN records of a chain need the end point and the S0
// prefix of segments handled by other lanes (or chunks): for groups of up to
// EMIT_STAGE segments the warp first stages them in shared memory, so the
// per-level SPAN emission reads shared memory instead of a chain of global loads.
// Per emitted segment the warp writes its hot records and one 24-B CopyRec
// (consecutive lanes: coalesced); the translation-invariant cold data of the
// segment was written once by K1 (BaseCold), whatever the number of copies.
#ifndef EMIT_WARPS
#define EMIT_WARPS 4
#endif
#ifndef EMIT_STAGE
#define EMIT_STAGE 128
#endif
#ifndef EMIT_MINB
#define EMIT_MINB 8
#endif
template <typename R>
__global__ void __launch_bounds__(32 * EMIT_WARPS, EMIT_MINB) k_emit(int32_t n_groups, const PlanGroup *__restrict__ groups,
                       const int32_t *__restrict__ loop_off,
                       const int32_t *__restrict__ loop_face, const uint8_t *__restrict__ face_per,
                       const double *__restrict__ face_dom, const double2 *__restrict__ lsta,
                       const double *__restrict__ s0, const int32_t *__restrict__ inv, const int2 *__restrict__ shift,
                       const uint8_t *__restrict__ brk,
                       const int2 *__restrict__ chain, const double *__restrict__ s0pre,
                       const double2 *__restrict__ lend,
                       const LoopInfo *__restrict__ info, double rel, Hot<R> *__restrict__ hot,
                       CopyRec *__restrict__ copy, int32_t n_rec_total, int32_t n_copy_total) {
  const int g = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (g >= n_groups) return;
  const PlanGroup G = groups[g];
  const int l = G.loop;
  const int f = loop_face[l];
  const int pu = face_per[f] & 1, pv = (face_per[f] >> 1) & 1;
  const double Tu = face_dom[4 * f + 1], Tv = face_dom[4 * f + 3];
  const LoopInfo I = info[l];
  const uint32_t fa = (G.flags & PF_ANGLE) ? F_ANGLE : 0u;
  // lsta / lend hold the LIFTED end points written by k_lift (lat(x, k_s, T)
  // per segment); translated coordinate of this group's copy:
  auto TX = [&](double x) { return pu ? lat(x, G.ku, Tu) : x; };
  auto TY = [&](double y) { return pv ? lat(y, G.kv, Tv) : y; };
  if (G.kind == G_LINE) {
    // omega(p, L) for the line through beta_0 along the extension vector (Eq. 5)
    if (lane == 0) {
      const double bx = TX(I.sx), by = TY(I.sy);
      if (I.cu != 0 && I.cv != 0) {                                    // general class: slanted line
        put_rec<R>(hot, G.rec_off, bx, by, 0.0, sline_meta(I.cu, I.cv));
        return;
      }
      uint32_t meta = K_LINE;
      double c;
      if (I.cu != 0) { c = by; if (I.cu > 0) meta |= F_GE; }          // v = (+-T,0): left iff p.v >=/<= c
      else { c = bx; meta |= F_AXISV; if (I.cv < 0) meta |= F_GE; }   // v = (0,+-T): left iff p.u <=/>= c
      put_rec<R>(hot, G.rec_off, c, 0.0, 0.0, meta);
    }
    return;
  }
  const int cull = (G.flags & PF_CULL) ? 1 : 0;
  if (cull && lane == 0) {
    const double xmin = TX(I.bb[0]) - G.M, xmax = TX(I.bb[2]) + G.M;
    const double ymin = TY(I.bb[1]) - G.M, ymax = TY(I.bb[3]) + G.M;
    put_group<R>(hot, G.rec_off, xmin, ymin, xmax, ymax, K_GROUP | ((uint32_t)(G.nrec - 1) << 8));
  }
  const int s0_ = loop_off[l], s1 = loop_off[l + 1];
  const int r_first = G.rec_off + cull + 1;              // first record after GROUP? and MOVE
  const bool tree = (G.flags & PF_TREE) != 0;
  const bool omit_root = tree && (G.flags & PF_OMIT_ROOT) != 0;
  __shared__ double2 s_end[EMIT_WARPS][EMIT_STAGE];      // translated lifted end points
  __shared__ double s_pre[EMIT_WARPS][EMIT_STAGE];       // S0 prefix sums
  const int wib = (threadIdx.x >> 5);
  const bool staged = tree && (s1 - s0_) <= EMIT_STAGE;
  if (staged) {
    for (int s = s0_ + lane; s < s1; s += 32) {
      const double2 le = lend[s];
      s_end[wib][s - s0_] = make_double2(TX(le.x), TY(le.y));
      s_pre[wib][s - s0_] = s0pre[s];
    }
    __syncwarp();
  }
  // fp64 records: spans of the conservative fp32 filter
  auto filter_span = [&](double S) {
    return (sizeof(R) == 8) ? (S * (1.0 + 0x1p-17) + G.M * 0x1p24) * (1.0 + 0x1p-17) : S * (1.0 + rel) + G.M;
  };
  int carry = 0;                                         // breaks before this chunk
  for (int base = s0_; base < s1; base += 32) {
    const int s = base + lane;
    const bool in = s < s1;
    const bool bk = in && s > s0_ && brk[s];
    const unsigned bm = __ballot_sync(0xffffffffu, bk);
    const int nb = carry + __popc(bm & ((2u << lane) - 1u));   // breaks in (s0, s]
    carry += __popc(bm);
    if (!in) continue;
    const int idx = s - s0_;
    const double2 e0 = lsta[s], e1 = lend[s];             // lifted end points (K2a)
    const double px0 = TX(e0.x), py0 = TY(e0.y), pxn = TX(e1.x), pyn = TY(e1.y);
    int r;
    if (!tree) {
      r = r_first + idx + nb;
      if (s == s0_) put_rec<R>(hot, r - 1, px0, py0, 0.0, K_MOVE | fa);
      else if (bk) put_rec<R>(hot, r - 1, px0, py0, 0.0, K_MOVEG | fa);
    } else {
      // path hierarchy: each chain of m segments becomes a pre-order
      // binary tree of 2m-1 records (SPAN nodes over segment ranges, SEG leaves);
      // chain c starts at record r_first + 2 * (its first segment index)
      const int2 ch = chain[s];                          // (chain start idx, chain length)
      const int j = idx - ch.x;
      int a = 0, bnd = ch.y - 1, off = r_first + 2 * ch.x;
      if (j == 0) {
        if (s == s0_) put_rec<R>(hot, off - 1, px0, py0, 0.0, K_MOVE | fa);
        else put_rec<R>(hot, off - 1, px0, py0, 0.0, K_MOVEG | fa);
      }
      int depth = 0;
      const int omit_k = omit_root ? OMIT_LEVELS : 0;    // closed loop: no top SPAN levels
      while (a < bnd) {
        const int mid = (a + bnd) >> 1;
        if (depth < omit_k) {                            // omitted level: no record
          if (j <= mid) bnd = mid;
          else { off += tree_recs(mid - a + 1, omit_k - depth - 1); a = mid + 1; }
          ++depth;
          continue;
        }
        ++depth;
        if (j == a) {
          // SPAN over chain segments [a, bnd]: foci = run ends, span = sum of S0
          const int se = s0_ + ch.x + bnd;               // last segment of the run
          const int sa = s0_ + ch.x + a;
          double ex, ey, sum;
          if (staged) {
            const double2 le = s_end[wib][se - s0_];
            ex = le.x; ey = le.y;
            sum = s_pre[wib][se - s0_] - (sa > s0_ ? s_pre[wib][sa - 1 - s0_] : 0.0);
          } else {
            const double2 le = lend[se];                 // its lifted end point (K2a)
            ex = TX(le.x); ey = TY(le.y);
            sum = s0pre[se] - (sa > s0_ ? s0pre[sa - 1] : 0.0);
          }
          const int sub = 2 * (bnd - a + 1) - 2;          // records of the subtree after the SPAN
          WN_DCHECK(off >= G.rec_off && off + sub < G.rec_off + G.nrec);
          put_rec<R>(hot, off, ex, ey, filter_span(sum), K_SPAN | fa | ((uint32_t)sub << 8));
        }
        if (j <= mid) { bnd = mid; off += 1; }
        else { off += 1 + (2 * (mid - a + 1) - 1); a = mid + 1; }
      }
      r = off;
    }
    // Root span (Eq. 1, R9) with the R5 margin.  fp64 records: the span of the
    // conservative fp32 filter, S0 (1 + 2^-17) + 2^-16 scale (scale = M 2^40),
    // and the filter's (1 - 2^-18) error shrink folded in as a further
    // (1 + 2^-17); fp32 records: S0 (1 + 2^-17) + M32.
    WN_DCHECK(r >= G.rec_off && r < G.rec_off + G.nrec && r < n_rec_total && G.cold_off + idx < n_copy_total);
    put_rec<R>(hot, r, pxn, pyn, filter_span(s0[s]), K_SEG | fa | ((uint32_t)(G.cold_local + idx) << 8));
    // the copy record: base segment, target face, lift shift, copy translate
    const int2 k = shift[s];
    CopyRec cr;
    cr.s = inv[s];
    cr.face = G.face;
    cr.ksu = pu ? k.x : 0;
    cr.ksv = pv ? k.y : 0;
    cr.ku = pu ? G.ku : 0;
    cr.kv = pv ? G.kv : 0;
    copy[G.cold_off + idx] = cr;
  }
  if (lane == 0) {
    int r = tree ? G.rec_off + cull + 1 + tree_recs(s1 - s0_, omit_root ? OMIT_LEVELS : 0)
                 : r_first + (s1 - s0_) + carry;
    if (G.flags & PF_TAIL_CLOSEG) put_rec<R>(hot, r++, 0.0, 0.0, 0.0, K_CLOSEG | fa);
    if (G.flags & PF_TAIL_XCH) put_rec<R>(hot, r++, 0.0, 0.0, 0.0, K_XCH | fa);
    if (G.flags & PF_TAIL_NCH) put_rec<R>(hot, r++, 0.0, 0.0, 0.0, K_NCH | fa);
  }
}

// ---------------------------------------------------------------------------
// host planner
// ---------------------------------------------------------------------------
__host__ __device__ inline int group_nrec(int kind, int flags, const LoopInfo &I);

struct Plan {
  std::vector<PlanGroup> groups;
  std::vector<int32_t> rec_off;   // per target face + 1
  std::vector<int32_t> cold_off;
  void reserve(size_t ng, size_t nf) { groups.reserve(ng); rec_off.reserve(nf + 1); cold_off.reserve(nf + 1); }
  // keep capacity (pages stay mapped across builds: page faults dominated the host plan)
  void clear() {
    groups.clear(); rec_off.clear(); cold_off.clear();
    n_lines = n_cull = 0; recs = colds = 0; face_rec0 = face_cold0 = 0; cur_face = -1;
  }
  int64_t n_lines = 0, n_cull = 0;
  int32_t recs = 0, colds = 0;
  int32_t face_rec0 = 0, face_cold0 = 0;
  int cur_face = -1;

  void begin_face(int f) {
    cur_face = f;
    face_rec0 = recs;
    face_cold0 = colds;
    rec_off.push_back(recs);
    cold_off.push_back(colds);
  }
  void end() {
    rec_off.push_back(recs);
    cold_off.push_back(colds);
  }
  void add(int kind, int flags, int loop, int ku, int kv, const LoopInfo &I, double M) {
    PlanGroup G;
    G.kind = kind;
    G.flags = flags;
    G.loop = loop;
    G.ku = ku;
    G.kv = kv;
    G.rec_off = recs;
    G.cold_off = colds;
    G.cold_local = colds - face_cold0;
    G.face = cur_face;
    G.M = M;
    int nrec;
    if (kind == G_LINE) {
      nrec = 1;
      ++n_lines;
    } else {
      // flat: MOVE + nseg SEG + nbrk MOVEG; tree: MOVE + sum_c (2 m_c - 1) + nbrk = 2 nseg
      nrec = group_nrec(kind, flags, I);
      colds += I.nseg;
      if (flags & PF_CULL) ++n_cull;
    }
    G.nrec = nrec;
    recs += nrec;
    groups.push_back(G);
  }
};

__host__ __device__ inline int gcd_i(int a, int b) {
  a = a < 0 ? -a : a;
  b = b < 0 ? -b : b;
  while (b) { int t = a % b; a = b; b = t; }
  return a;
}

// lattice translates k with [lo + k T, hi + k T] meeting [t0 - m, t0 + T + m]
__host__ __device__ inline void k_range(double lo, double hi, double t0, double T, double m, int &k0, int &k1) {
  k0 = (int)ceil((t0 - m - hi) / T) - 1;
  k1 = (int)floor((t0 + T + m - lo) / T) + 1;
  // tighten exactly (the +-1 guards the division rounding)
  while (k0 <= k1 && !(lo + k0 * T <= t0 + T + m && hi + k0 * T >= t0 - m)) ++k0;
  while (k1 >= k0 && !(lo + k1 * T <= t0 + T + m && hi + k1 * T >= t0 - m)) --k1;
}

struct FaceCtx {
  uint8_t per;
  double u0, Tu, v0, Tv;
  double M;
  bool angle;
};

// hot records of one planned group (must match k_emit's layout)
__host__ __device__ inline int group_nrec(int kind, int flags, const LoopInfo &I) {
  if (kind == G_LINE) return 1;
  // flat: MOVE + nseg SEG + nbrk MOVEG; tree: MOVE + sum_c (2 m_c - 1) + nbrk = 2 nseg,
  // minus the omitted top SPAN levels of a closed single-chain loop
  return ((flags & PF_CULL) ? 1 : 0) + ((flags & PF_TREE) ? 2 * I.nseg : 1 + I.nseg + I.nbrk) -
         ((flags & PF_OMIT_ROOT) ? tree_internal_top(I.nseg, OMIT_LEVELS) : 0) +
         ((flags & (PF_TAIL_CLOSEG | PF_TAIL_XCH | PF_TAIL_NCH)) ? 1 : 0);
}

// group flags for a closed / copy group
__host__ __device__ inline int loop_flags(const LoopInfo &I, bool angle, bool copy, bool tree) {
  int fl = (angle ? PF_ANGLE : 0) | (tree ? PF_TREE : 0);
  if (copy) {
    fl |= angle ? PF_TAIL_NCH : PF_TAIL_XCH;
    if (I.nbrk == 0) fl |= PF_CULL;
  } else {
    const bool closed = I.closed && I.nbrk == 0;
    if (closed) fl |= PF_CULL;
    else if (!angle) fl |= PF_TAIL_CLOSEG;
    // a closed loop is one chain whose ends coincide: the root SPAN's ellipse is
    // the circle of radius sum(S0)/2 around its start -- it (almost) never
    // prunes, so the tree starts at the root's two children
    if (closed && tree) fl |= PF_OMIT_ROOT;
  }
  return fl;
}

__host__ __device__ inline double tile_margin(const FaceCtx &C) {
  return 1e-9 * (1.0 + fabs(C.u0) + C.Tu + fabs(C.v0) + C.Tv);
}

// contractible loop in a (uni/bi/non-)periodic face: every translate meeting the tile
template <class S>
__host__ __device__ void plan_contractible(S &P, int l, const LoopInfo &I, const FaceCtx &C, bool tree,
                                           bool no_cull = false) {
  int fl = loop_flags(I, C.angle, false, tree);
  if (no_cull) fl &= ~PF_CULL;
  int i0 = 0, i1 = 0, j0 = 0, j1 = 0;
  const double m = tile_margin(C);
  if (C.per & 1) k_range(I.bb[0], I.bb[2], C.u0, C.Tu, m, i0, i1);
  if (C.per & 2) k_range(I.bb[1], I.bb[3], C.v0, C.Tv, m, j0, j1);
  for (int i = i0; i <= i1; ++i)
    for (int j = j0; j <= j1; ++j) P.add(G_LOOP, fl, l, i, j, I, C.M);
}

// non-contractible loop along axis a (0 = u, 1 = v) at transverse translate jt:
// copies (Eq. 5 rewritten with chords tiling L) meeting the tile
template <class S>
__host__ __device__ void plan_extended_copies(S &P, int l, const LoopInfo &I, const FaceCtx &C, int axis, int jt,
                                              bool transverse_cull_tile, bool tree) {
  const int fl = loop_flags(I, C.angle, true, tree);
  const double m = tile_margin(C);
  int k0, k1;
  if (axis == 0) k_range(I.bb[0], I.bb[2], C.u0, C.Tu, m, k0, k1);
  else k_range(I.bb[1], I.bb[3], C.v0, C.Tv, m, k0, k1);
  if (transverse_cull_tile) {
    // bi-periodic: the transverse translate must also meet the tile
    const double lo = axis == 0 ? I.bb[1] + jt * C.Tv : I.bb[0] + jt * C.Tu;
    const double hi = axis == 0 ? I.bb[3] + jt * C.Tv : I.bb[2] + jt * C.Tu;
    const double t0 = axis == 0 ? C.v0 : C.u0, T = axis == 0 ? C.Tv : C.Tu;
    if (!(lo <= t0 + T + m && hi >= t0 - m)) return;
  }
  for (int k = k0; k <= k1; ++k) {
    if (axis == 0) P.add(G_COPY, fl, l, k, jt, I, C.M);
    else P.add(G_COPY, fl, l, jt, k, I, C.M);
  }
}

// ---- general bi-periodic classes (p,q), p,q != 0 (Prop. 2; Eq. 8) ----
// Band coordinate nu(x) = p*y/Tv - q*x/Tu: the lattice translate (i Tu, j Tv)
// shifts it by m = p*j - q*i, and translates with equal m differ by multiples
// of the extension vector v = (p Tu, q Tv), i.e. give the same extended curve.
// So the extended curves gamma_{r,s} of Eq. (8) are indexed by the integer m
// (gcd = 1: every m occurs once over r in [0,|p|), s in Z).
__host__ __device__ inline double band_nu(int p, int q, const FaceCtx &C, double x, double y) {
  return (double)p * y / C.Tv - (double)q * x / C.Tu;
}
// one translate (i, j) with p*j - q*i = m
__host__ __device__ inline void band_rep(int p, int q, int m, int &i, int &j) {
  int x0 = 0, y0 = 0;
  if (p == 0) {
    x0 = -q;                                    // q = +-1
  } else {
    const int ap = p < 0 ? -p : p;
    for (int x = 0; x < ap; ++x)
      if ((1 + q * x) % p == 0) { x0 = x; y0 = (1 + q * x) / p; break; }
  }
  i = m * x0;
  j = m * y0;
}
__host__ __device__ inline void box_nu(const double *bb, int p, int q, const FaceCtx &C, int i, int j, double &lo,
                                       double &hi) {
  lo = INFINITY; hi = -INFINITY;
  for (int c = 0; c < 4; ++c) {
    const double nu = band_nu(p, q, C, bb[(c & 1) ? 2 : 0] + i * C.Tu, bb[(c & 2) ? 3 : 1] + j * C.Tv);
    lo = fmin(lo, nu); hi = fmax(hi, nu);
  }
}
__host__ __device__ inline int floor_div(int a, int b) { int d = a / b; return (a % b != 0 && ((a < 0) != (b < 0))) ? d - 1 : d; }
__host__ __device__ inline int ceil_div(int a, int b) { return -floor_div(-a, b); }
// k with lo <= t + k d <= hi, intersected into [klo, khi]
__host__ __device__ inline void k_restrict(int t, int d, int lo, int hi, int &klo, int &khi) {
  if (d > 0) { klo = max(klo, ceil_div(lo - t, d)); khi = min(khi, floor_div(hi - t, d)); }
  else if (d < 0) { klo = max(klo, ceil_div(hi - t, d)); khi = min(khi, floor_div(lo - t, d)); }
  else if (t < lo || t > hi) khi = klo - 1;
}
// copies (loop + (ti + k p, tj + k q) tiles) of one extended curve whose box meets the tile
template <class S>
__host__ __device__ void plan_band_copies(S &P, int l, const LoopInfo &I, const FaceCtx &C, int p, int q, int ti,
                                          int tj, bool tree) {
  const int fl = loop_flags(I, C.angle, true, tree);
  const double m = tile_margin(C);
  int a0, a1, b0, b1;
  k_range(I.bb[0], I.bb[2], C.u0, C.Tu, m, a0, a1);   // u-translates meeting the tile
  k_range(I.bb[1], I.bb[3], C.v0, C.Tv, m, b0, b1);   // v-translates meeting the tile
  if (a0 > a1 || b0 > b1) return;
  int klo = -(1 << 29), khi = 1 << 29;
  k_restrict(ti, p, a0, a1, klo, khi);
  k_restrict(tj, q, b0, b1, klo, khi);
  for (int k = klo; k <= khi; ++k) P.add(G_COPY, fl, l, ti + k * p, tj + k * q, I, C.M);
}
// Eq. 8 for a general pair (alpha, beta-bar = beta + rep(mb)): every band m
// whose strip or copies can meet the base tile
template <class S>
__host__ __device__ void plan_general_pair(S &P, int l, const LoopInfo &I, int lb, const LoopInfo &Ib, int mb,
                                           const FaceCtx &C, bool tree) {
  const int p = I.cu, q = I.cv;
  int bi, bj;
  band_rep(p, q, mb, bi, bj);
  double alo, ahi, blo, bhi;
  box_nu(I.bb, p, q, C, 0, 0, alo, ahi);
  box_nu(Ib.bb, p, q, C, bi, bj, blo, bhi);
  const double na = band_nu(p, q, C, I.sx, I.sy), nb = band_nu(p, q, C, Ib.sx + bi * C.Tu, Ib.sy + bj * C.Tv);
  const double lo = fmin(fmin(alo, blo), fmin(na, nb)), hi = fmax(fmax(ahi, bhi), fmax(na, nb));
  const double mt = tile_margin(C);
  double tlo = INFINITY, thi = -INFINITY;
  for (int c = 0; c < 4; ++c) {
    const double nu = band_nu(p, q, C, (c & 1) ? C.u0 + C.Tu + mt : C.u0 - mt, (c & 2) ? C.v0 + C.Tv + mt : C.v0 - mt);
    tlo = fmin(tlo, nu); thi = fmax(thi, nu);
  }
  const double sl = 1e-6;                       // slack: extra bands only cost records
  const int m0 = (int)floor(tlo - hi - sl) - 1, m1 = (int)ceil(thi - lo + sl) + 1;
  for (int m = m0; m <= m1; ++m) {
    int i, j;
    band_rep(p, q, m, i, j);
    // omega(p, L_alpha) + omega(p, L_beta) cancel unless the strip meets the tile
    if (fmin(na, nb) + m <= thi + sl && fmax(na, nb) + m >= tlo - sl) {
      P.add(G_LINE, 0, l, i, j, I, C.M);
      P.add(G_LINE, 0, lb, bi + i, bj + j, Ib, C.M);
    }
    plan_band_copies(P, l, I, C, p, q, i, j, tree);
    plan_band_copies(P, lb, Ib, C, p, q, bi + i, bj + j, tree);
  }
}

// the groups of one (validated, paired) face
template <class S>
__host__ __device__ void plan_face(S &P, const LoopInfo *L, int l0, int l1, const FaceCtx &C,
                                   const int *pair_beta, const int *pair_s, bool tree) {
  // Non-periodic face: the loop whose box holds every other loop's box (the
  // outer boundary) gets no cull header -- its box is the face's query box, so
  // the header would pass for (nearly) every query and only cost an iteration
  // (a query outside it prunes at the loop's first hierarchy level instead)
  int outer = -1;
  if (C.per == 0) {
    double x0 = INFINITY, y0 = INFINITY, x1 = -INFINITY, y1 = -INFINITY;
    for (int l = l0; l < l1; ++l) {
      if (L[l].nseg == 0) continue;
      x0 = fmin(x0, L[l].bb[0]); y0 = fmin(y0, L[l].bb[1]);
      x1 = fmax(x1, L[l].bb[2]); y1 = fmax(y1, L[l].bb[3]);
    }
    for (int l = l0; l < l1 && outer < 0; ++l)
      if (L[l].nseg && L[l].bb[0] == x0 && L[l].bb[1] == y0 && L[l].bb[2] == x1 && L[l].bb[3] == y1) outer = l;
  }
  for (int l = l0; l < l1; ++l) {
    const LoopInfo &I = L[l];
    if (I.nseg == 0) continue;
    if (C.per == 0 || (I.cu == 0 && I.cv == 0)) {
      plan_contractible(P, l, I, C, tree, l == outer);
      continue;
    }
    const int axis = (I.cu != 0) ? 0 : 1;
    if (C.per != 3) {
      // uni-periodic non-contractible loop: omega(p,L) + copies (Eq. 5)
      P.add(G_LINE, 0, l, 0, 0, I, C.M);
      plan_extended_copies(P, l, I, C, axis, 0, false, tree);
      continue;
    }
    // bi-periodic: alpha loops drive Eq. 8 for their pair; beta loops are emitted with them
    if (!pair_beta || pair_beta[l] < 0) continue;
    const int lb = pair_beta[l];
    const int sb = pair_s[l];
    const LoopInfo &Ib = L[lb];
    if (I.cu != 0 && I.cv != 0) {
      plan_general_pair(P, l, I, lb, Ib, sb, C, tree);
      continue;
    }
    const int tax = axis == 0 ? 1 : 0;
    const double Tt = tax ? C.Tv : C.Tu, t0 = tax ? C.v0 : C.u0;
    const double m = tile_margin(C);
    // transverse window: every band offset j whose lines or copies can meet the tile
    const double ca = tax ? I.sy : I.sx, cb = (tax ? Ib.sy : Ib.sx) + sb * Tt;
    const double lo = fmin(fmin(ca, cb), fmin(tax ? I.bb[1] : I.bb[0], (tax ? Ib.bb[1] : Ib.bb[0]) + sb * Tt));
    const double hi = fmax(fmax(ca, cb), fmax(tax ? I.bb[3] : I.bb[2], (tax ? Ib.bb[3] : Ib.bb[2]) + sb * Tt));
    int j0, j1;
    k_range(lo, hi, t0, Tt, m, j0, j1);
    for (int j = j0; j <= j1; ++j) {
      // Eq. 8 band j: omega(p, L_alpha) + omega(p, L_beta) only when the strip meets the tile
      const double la_c = ca + j * Tt, lb_c = cb + j * Tt;
      if (fmin(la_c, lb_c) <= t0 + Tt + m && fmax(la_c, lb_c) >= t0 - m) {
        if (axis == 0) { P.add(G_LINE, 0, l, 0, j, I, C.M); P.add(G_LINE, 0, lb, 0, sb + j, Ib, C.M); }
        else { P.add(G_LINE, 0, l, j, 0, I, C.M); P.add(G_LINE, 0, lb, sb + j, 0, Ib, C.M); }
      }
      plan_extended_copies(P, l, I, C, axis, j, true, tree);
      plan_extended_copies(P, lb, Ib, C, axis, sb + j, true, tree);
    }
  }
}

__host__ __device__ inline double face_margin(const LoopInfo *L, int l0, int l1, const FaceCtx &C, bool fp32) {
  const double ext = ((C.per & 1) ? 2 * C.Tu : 0.0) + ((C.per & 2) ? 2 * C.Tv : 0.0);
  double s = 1.0 + fabs(C.u0) + fabs(C.v0) + ext;
  for (int l = l0; l < l1; ++l)
    for (int k = 0; k < 4; ++k) s = fmax(s, 1.0 + fabs(L[l].bb[k]) + ext);
  return fp32 ? ldexp(s, -17) : ldexp(s, -40);
}

// face context from the stored periodicity / domain (non-periodic axes zeroed)
__host__ __device__ inline FaceCtx face_ctx(uint8_t per, const double *dom, bool angle) {
  FaceCtx C;
  C.per = per & 3;
  C.u0 = dom[0]; C.Tu = dom[1]; C.v0 = dom[2]; C.Tv = dom[3];
  if (!(C.per & 1)) { C.u0 = 0; C.Tu = 0; }
  if (!(C.per & 2)) { C.v0 = 0; C.Tv = 0; }
  C.angle = angle;
  C.M = 0.0;
  return C;
}

// topology validation of one face (Prop. 1; R12-R16): WN_FACE_* code;
// *needp = 1 when the face's non-contractible loops must be paired (Algs. 7-9)
__host__ __device__ inline int face_validate(const LoopInfo *L, int l0, int l1, const FaceCtx &C, bool strict,
                                             int *needp) {
  int st = WN_FACE_OK;
  *needp = 0;
  int cp = 0, cq = 0, nA = 0, nB = 0;
  for (int l = l0; l < l1; ++l) {
    const LoopInfo &I = L[l];
    if (I.err) st = WN_FACE_GEOM;
    if (I.nseg == 0 || (I.cu == 0 && I.cv == 0)) continue;
    if (C.per == 1 && abs(I.cu) > 1) st = WN_FACE_B1;
    if (C.per == 2 && abs(I.cv) > 1) st = WN_FACE_B1;
    if (gcd_i(I.cu, I.cv) != 1 && !st) st = WN_FACE_CLASS;
    if (cp == 0 && cq == 0) { cp = I.cu; cq = I.cv; }
    if (I.cu == cp && I.cv == cq) ++nA;
    else if (I.cu == -cp && I.cv == -cq) ++nB;
    else if (!st) st = WN_FACE_CLASS;
  }
  if (st) return st;
  if (nA != nB && (strict || C.per == 3)) return WN_FACE_UNBALANCED;
  if (C.per == 3 && nA > 0) *needp = 1;
  return WN_FACE_OK;
}

// ---------------------------------------------------------------------------
// K2b on the device: one thread per face validates it, derives its margin and
// plans its groups twice -- a counting pass, a scan, and a filling pass that
// writes the PlanGroups where k_emit reads them.  The host only reads a small
// summary (totals for the record allocations, validation outcome).
// ---------------------------------------------------------------------------
struct BuildSummary {
  int bad, needp, geom, unsup, toobig, maxr;
  unsigned long long first_bad;   // (face << 32) | code, minimum over bad faces
  int tot_g, tot_r, tot_c, pad;
  unsigned long long lines, cull;
  unsigned long long copies, bands;   // extended-copy groups; Eq. 8 bands (line pairs of bi-periodic faces)
  int csr_bad;                        // loop / face CSR offsets not a valid CSR (k_csr_check)
  unsigned dom_bad;                   // min over faces of (face << 1 | axis) with a bad period, else ~0
};

// Input validation on the device (the host reads only the summary): CSR
// offsets start at 0, end at the element count and never decrease; periodic
// axes have a finite start and a finite period > 0.
__global__ void k_csr_check(int32_t n_loops, int32_t n_faces, int32_t n_segs, const int32_t *__restrict__ lso,
                            const int32_t *__restrict__ flo, const uint8_t *__restrict__ per,
                            const double *__restrict__ dom, BuildSummary *__restrict__ sum) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  bool bad = false;
  if (i <= n_loops) {
    const int a = lso[i];
    if (i == 0 && a != 0) bad = true;
    if (i == n_loops && a != n_segs) bad = true;
    if (i < n_loops && a > lso[i + 1]) bad = true;
  }
  if (i <= n_faces) {
    const int a = flo[i];
    if (i == 0 && a != 0) bad = true;
    if (i == n_faces && a != n_loops) bad = true;
    if (i < n_faces && a > flo[i + 1]) bad = true;
  }
  if (bad) atomicOr(&sum->csr_bad, 1);
  if (i < n_faces) {
    const uint8_t pf = per[i];
    const double *d = dom + 4 * i;
    if ((pf & 1) && !(isfinite(d[0]) && isfinite(d[1]) && d[1] > 0)) atomicMin(&sum->dom_bad, ((unsigned)i << 1) | 0u);
    if ((pf & 2) && !(isfinite(d[2]) && isfinite(d[3]) && d[3] > 0)) atomicMin(&sum->dom_bad, ((unsigned)i << 1) | 1u);
  }
}

struct CountSink {
  int ng = 0, recs = 0, colds = 0, lines = 0, cull = 0, copies = 0;
  __device__ void add(int kind, int flags, int, int, int, const LoopInfo &I, double) {
    ++ng;
    recs += group_nrec(kind, flags, I);
    if (kind == G_LINE) ++lines;
    else {
      if (kind == G_COPY) ++copies;
      colds += I.nseg;
      if (flags & PF_CULL) ++cull;
    }
  }
};

struct FillSink {
  PlanGroup *out;
  int face, recs, colds, cold0;
  __device__ void add(int kind, int flags, int loop, int ku, int kv, const LoopInfo &I, double M) {
    PlanGroup G;
    G.kind = kind;
    G.flags = flags;
    G.loop = loop;
    G.ku = ku;
    G.kv = kv;
    G.rec_off = recs;
    G.cold_off = colds;
    G.cold_local = colds - cold0;
    G.nrec = group_nrec(kind, flags, I);
    G.face = face;
    G.M = M;
    *out++ = G;
    recs += G.nrec;
    if (kind != G_LINE) colds += I.nseg;
  }
};

__global__ void k_plan_count(int32_t n_faces, int32_t n_loops, const int32_t *__restrict__ flo,
                             const uint8_t *__restrict__ per,
                             const double *__restrict__ dom, const LoopInfo *__restrict__ L, int angle, int strict,
                             int tree, int fp32, const int *__restrict__ pair_beta, const int *__restrict__ pair_s,
                             int32_t *__restrict__ status, uint8_t *__restrict__ fper, double *__restrict__ fdom,
                             double *__restrict__ fM, float4 *__restrict__ fbox, int4 *__restrict__ cnt,
                             uint32_t *__restrict__ okey,
                             int32_t *__restrict__ oval, BuildSummary *__restrict__ sum) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= n_faces) return;
  const int l0 = min(max(flo[f], 0), n_loops), l1 = min(max(flo[f + 1], l0), n_loops);   // clamped (host-validated)
  FaceCtx C = face_ctx(per[f], dom + 4 * f, angle != 0);
  C.M = face_margin(L, l0, l1, C, fp32 != 0);
  int needp = 0;
  const int st = face_validate(L, l0, l1, C, strict != 0, &needp);
  status[f] = st;
  fper[f] = C.per;
  fdom[4 * f] = C.u0; fdom[4 * f + 1] = C.Tu; fdom[4 * f + 2] = C.v0; fdom[4 * f + 3] = C.Tv;
  fM[f] = C.M;
  {
    // box of the queries that can be inside: the loops' boxes, the base tile
    // on periodic axes (queries are reduced into it); only a regrouping key
    float x0 = INFINITY, y0 = INFINITY, x1 = -INFINITY, y1 = -INFINITY;
    for (int l = l0; l < l1; ++l) {
      if (L[l].nseg == 0) continue;
      x0 = fminf(x0, (float)L[l].bb[0]); y0 = fminf(y0, (float)L[l].bb[1]);
      x1 = fmaxf(x1, (float)L[l].bb[2]); y1 = fmaxf(y1, (float)L[l].bb[3]);
    }
    if (C.per & 1) { x0 = (float)C.u0; x1 = (float)(C.u0 + C.Tu); }
    if (C.per & 2) { y0 = (float)C.v0; y1 = (float)(C.v0 + C.Tv); }
    if (!(x1 > x0) || !(y1 > y0) || !isfinite(x1 - x0) || !isfinite(y1 - y0)) x0 = y0 = x1 = y1 = 0.f;
    fbox[f] = make_float4(x0, y0, x1, y1);
  }
  CountSink S;
  if (st) {
    atomicOr(&sum->bad, 1);
    if (st == WN_FACE_GEOM) atomicOr(&sum->geom, 1);
    if (st == WN_FACE_GENERAL_PQ) atomicOr(&sum->unsup, 1);
    atomicMin(&sum->first_bad, ((unsigned long long)f << 32) | (unsigned)st);
  } else if (needp && !pair_beta) {
    atomicOr(&sum->needp, 1);
  } else {
    plan_face(S, L, l0, l1, C, pair_beta, pair_s, tree != 0);
    if (S.lines) atomicAdd(&sum->lines, (unsigned long long)S.lines);
    if (S.cull) atomicAdd(&sum->cull, (unsigned long long)S.cull);
    if (S.copies) atomicAdd(&sum->copies, (unsigned long long)S.copies);
    if (C.per == 3 && S.lines) atomicAdd(&sum->bands, (unsigned long long)(S.lines / 2));
    if (S.recs >= (1 << 24) || S.colds >= (1 << 22)) atomicOr(&sum->toobig, 1);
    atomicMax(&sum->maxr, S.recs);
  }
  cnt[f] = make_int4(S.ng, S.recs, S.colds, 0);
  okey[f] = 0xffffffffu - (uint32_t)S.recs;   // ascending key = descending record count
  oval[f] = f;
}

// exclusive scans of the per-face (groups, records, colds) -- one block
constexpr int PLAN_SCAN_T = 1024;
__global__ void __launch_bounds__(PLAN_SCAN_T) k_plan_scan(int32_t n_faces, const int4 *__restrict__ cnt,
                                                           int4 *__restrict__ off, int32_t *__restrict__ rec_off,
                                                           int32_t *__restrict__ cold_off,
                                                           BuildSummary *__restrict__ sum) {
  __shared__ long long s_part[3][PLAN_SCAN_T];
  const int t = threadIdx.x;
  const int per_t = (n_faces + PLAN_SCAN_T - 1) / PLAN_SCAN_T;
  const int f0 = min(n_faces, t * per_t), f1 = min(n_faces, f0 + per_t);
  long long a = 0, r = 0, c = 0;
  for (int f = f0; f < f1; ++f) { a += cnt[f].x; r += cnt[f].y; c += cnt[f].z; }
  s_part[0][t] = a; s_part[1][t] = r; s_part[2][t] = c;
  __syncthreads();
  for (int o = 1; o < PLAN_SCAN_T; o <<= 1) {   // Hillis-Steele inclusive scan
    long long va = 0, vr = 0, vc = 0;
    if (t >= o) { va = s_part[0][t - o]; vr = s_part[1][t - o]; vc = s_part[2][t - o]; }
    __syncthreads();
    s_part[0][t] += va; s_part[1][t] += vr; s_part[2][t] += vc;
    __syncthreads();
  }
  long long ba = t ? s_part[0][t - 1] : 0, br = t ? s_part[1][t - 1] : 0, bc = t ? s_part[2][t - 1] : 0;
  for (int f = f0; f < f1; ++f) {
    off[f] = make_int4((int)ba, (int)br, (int)bc, 0);
    rec_off[f] = (int)br;
    cold_off[f] = (int)bc;
    ba += cnt[f].x; br += cnt[f].y; bc += cnt[f].z;
  }
  if (t == PLAN_SCAN_T - 1) {
    const long long ta = s_part[0][t], tr = s_part[1][t], tc = s_part[2][t];
    rec_off[n_faces] = (int)tr;
    cold_off[n_faces] = (int)tc;
    if (ta > INT32_MAX || tr > INT32_MAX || tc >= (1ll << 23) * 64) sum->toobig = 1;
    sum->tot_g = (int)ta;
    sum->tot_r = (int)tr;
    sum->tot_c = (int)tc;
  }
}

__global__ void k_plan_fill(int32_t n_faces, int32_t n_loops, const int32_t *__restrict__ flo,
                            const uint8_t *__restrict__ fper,
                            const double *__restrict__ fdom, const double *__restrict__ fM,
                            const LoopInfo *__restrict__ L, int angle, int tree, const int *__restrict__ pair_beta,
                            const int *__restrict__ pair_s, const int4 *__restrict__ off,
                            PlanGroup *__restrict__ groups) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= n_faces) return;
  FaceCtx C = face_ctx(fper[f], fdom + 4 * f, angle != 0);
  C.M = fM[f];
  const int4 o = off[f];
  FillSink S{groups + o.x, f, o.y, o.z, o.z};
  const int l0 = min(max(flo[f], 0), n_loops), l1 = min(max(flo[f + 1], l0), n_loops);
  plan_face(S, L, l0, l1, C, pair_beta, pair_s, tree != 0);
  WN_DCHECK(f + 1 >= n_faces || S.out == groups + off[f + 1].x);   // the fill pass wrote exactly the counted groups
}

}  // namespace wn

using namespace wn;

// ---------------------------------------------------------------------------
// pinned host staging (build-time transfers) and device buffers helper
// ---------------------------------------------------------------------------
namespace {
// Bump allocator over pinned host blocks; reset at the start of every build
// (each build ends with a stream synchronisation, so no copy is in flight).
struct PinnedArena {
  std::vector<std::pair<char *, size_t>> blocks;
  size_t blk = 0, off = 0;
  void reset() { blk = 0; off = 0; }
  void *get(size_t bytes) {
    bytes = (bytes + 255) & ~(size_t)255;
    while (blk < blocks.size() && off + bytes > blocks[blk].second) { ++blk; off = 0; }
    if (blk == blocks.size()) {
      size_t sz = std::max(bytes, (size_t)64 << 20);
      char *p = nullptr;
      if (cudaMallocHost((void **)&p, sz) != cudaSuccess) return nullptr;
      blocks.push_back({p, sz});
      off = 0;
    }
    void *r = blocks[blk].first + off;
    off += bytes;
    return r;
  }
};
PinnedArena g_pin;
std::mutex g_build_mu;
// The build returns without waiting for its device work: the pinned staging of
// one build stays in use until the event recorded after its last copy, which
// the next build waits on before reusing the arena (per device).
cudaEvent_t g_pin_ev[64] = {};
bool g_pin_pending[64] = {};
// per device: the auxiliary stream of the device planner and its fork/join events
cudaStream_t g_aux[64] = {};
// per device: K1's side streams and their fork / join events (launch_k1)
cudaStream_t g_k1s[64][3] = {};
cudaEvent_t g_k1ev[64][4] = {};
cudaEvent_t g_ev_lift[64] = {}, g_ev_plan[64] = {}, g_ev_fill[64] = {}, g_ev_k1[64] = {};
struct PinRelease {
  cudaEvent_t ev;
  bool *pending;
  cudaStream_t st;
  ~PinRelease() {
    if (cudaEventRecord(ev, st) == cudaSuccess) *pending = true;
  }
};

cudaError_t h2d(void *dst, const void *src, size_t bytes, cudaStream_t st) {
  if (!bytes) return cudaSuccess;
  void *s = g_pin.get(bytes);
  if (!s) return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st);
  memcpy(s, src, bytes);
  return cudaMemcpyAsync(dst, s, bytes, cudaMemcpyHostToDevice, st);
}

struct DevBuf {
  std::vector<void *> ptrs;
  cudaStream_t st = 0;
  ~DevBuf() {
    for (void *p : ptrs) cache_free(p, st);
  }
  template <typename T>
  cudaError_t alloc(T **p, size_t count) {
    cudaError_t e = cache_alloc((void **)p, sizeof(T) * (count ? count : 1), st);
    if (e == cudaSuccess) ptrs.push_back(*p);
    return e;
  }
};

void free_handle(wn_faces_t F) {
  if (!F) return;
  if (!F->k3_events.empty()) {   // unread timing survives the handle (wn_get_timing(NULL, ...))
    std::vector<K3Timing> ev;
    for (size_t i = 0; i < F->k3_events.size(); ++i)
      ev.push_back({F->k3_events[i].first, F->k3_mid[i], F->k3_events[i].second});
    orphan_timing(std::move(ev));
  }
  // stream-ordered frees on the legacy stream, after the handle's last use
  // (its build or its latest query, on whatever stream that ran)
  if (F->last_use) cudaStreamWaitEvent(0, F->last_use, 0);
  if (F->owns_cold && F->cold) cache_free(F->cold, 0);
  void *ps[] = {F->hot, F->copy, F->owns_cold ? (void *)F->inv : nullptr, F->face_rec_off, F->face_cold_off, F->face_order, F->face_dom,
                F->face_per, F->face_ok, F->face_M, F->face_box, F->counters};
  for (void *p : ps)
    if (p) cache_free(p, 0);
  if (F->last_use) cudaEventDestroy(F->last_use);
  if (F->ready) cudaEventDestroy(F->ready);
  delete F;
}

// Everything the emission (and the pairing probes) reads is library-owned:
// ctrl / w are the lifted copies written by k_lift, deg / lso / flo copies of
// the caller's arrays, per / dom the handle's face arrays.  The caller's
// buffers are read only by work that completes before wn_build_faces returns.
struct BuildCtx {
  int32_t n_faces, n_loops, n_segs;
  const int32_t *deg, *lso, *flo;
  const uint8_t *per;
  const double *dom;
  int32_t *coff, *loop_face;
  double *s0;       // per segment: root span S0 (K1, unmargined)
  int32_t *inv;     // per segment: its BaseCold record (position in K1's degree-sorted order)
  int2 *shift;      // per segment: lift shift (K2a)
  uint8_t *brk;
  int2 *chain;      // per segment: (chain start index within its loop, chain length)
  double *s0pre;    // per segment: prefix sum of root spans S0 along its loop
  double2 *lsta;    // per segment: lifted start point
  double2 *lend;    // per segment: lifted end point
  LoopInfo *info;
  cudaStream_t st;
};

// K1 launch, shared by wn_build_faces and wn_segment_prep: segments sorted by
// degree (3-bit radix sort), then one kernel per degree over its range of the
// sorted order, each with its own register budget (PREP_SPLIT CTAs per SM).
template <class Sink>
cudaError_t launch_k1(int32_t n_segs, const int32_t *deg, const int32_t *coff, const double *ctrl, const double *w,
                      const Sink &sink, uint8_t *serr, DevBuf &D, cudaStream_t st) {
  if (n_segs <= 0) return cudaSuccess;
  int32_t *d_iota = nullptr, *d_order = nullptr, *d_degs = nullptr;
  cudaError_t e;
  if ((e = D.alloc(&d_iota, n_segs)) != cudaSuccess) return e;
  if ((e = D.alloc(&d_order, n_segs)) != cudaSuccess) return e;
  if ((e = D.alloc(&d_degs, n_segs)) != cudaSuccess) return e;
  k_iota<<<(n_segs + 255) / 256, 256, 0, st>>>(n_segs, d_iota);
  size_t tmp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp, deg, d_degs, d_iota, d_order, n_segs, 0, 3, st);
  char *dt = nullptr;
  if ((e = D.alloc(&dt, tmp)) != cudaSuccess) return e;
  cub::DeviceRadixSort::SortPairs(dt, tmp, deg, d_degs, d_iota, d_order, n_segs, 0, 3, st);
  g_build_launches += 4;
  int32_t *d_bnd = nullptr;
  if ((e = D.alloc(&d_bnd, 9)) != cudaSuccess) return e;
  k_deg_bounds<<<(n_segs + 1 + 255) / 256, 256, 0, st>>>(n_segs, d_degs, d_bnd);
  const int pg = std::min((n_segs + 127) / 128, 148 * PREP_SPLIT);
  const size_t sm = Sink::kStaged ? 128 * sizeof(typename Sink::Rec) : 0;
#if K1_STREAMS
  // the degree kernels run concurrently on side streams (forked from / joined
  // back to `st`), so one kernel's last wave overlaps the next one's first
  int dev = 0;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  if (!g_k1s[dev][0]) {
    for (int i = 0; i < 3; ++i)
      if ((e = cudaStreamCreateWithFlags(&g_k1s[dev][i], cudaStreamNonBlocking)) != cudaSuccess) return e;
    for (int i = 0; i < 4; ++i)
      if ((e = cudaEventCreateWithFlags(&g_k1ev[dev][i], cudaEventDisableTiming)) != cudaSuccess) return e;
  }
  cudaStream_t *ss = g_k1s[dev];
  if ((e = cudaEventRecord(g_k1ev[dev][3], st)) != cudaSuccess) return e;
  for (int i = 0; i < 3; ++i)
    if ((e = cudaStreamWaitEvent(ss[i], g_k1ev[dev][3], 0)) != cudaSuccess) return e;
  k_prep_deg<5><<<pg, 128, sm, st>>>(d_bnd, deg, coff, ctrl, w, sink, serr, d_order);
  k_prep_deg<4><<<pg, 128, sm, ss[0]>>>(d_bnd, deg, coff, ctrl, w, sink, serr, d_order);
  k_prep_deg<3><<<pg, 128, sm, ss[1]>>>(d_bnd, deg, coff, ctrl, w, sink, serr, d_order);
  k_prep_deg<2><<<pg, 128, sm, ss[2]>>>(d_bnd, deg, coff, ctrl, w, sink, serr, d_order);
  k_prep_deg<1><<<pg, 128, sm, ss[2]>>>(d_bnd, deg, coff, ctrl, w, sink, serr, d_order);
  k_prep_bad<<<std::min((n_segs + 255) / 256, 148), 256, 0, st>>>(d_bnd, sink, serr, d_order);
  for (int i = 0; i < 3; ++i) {
    if ((e = cudaEventRecord(g_k1ev[dev][i], ss[i])) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(st, g_k1ev[dev][i], 0)) != cudaSuccess) return e;
  }
#else
  k_prep_deg<5><<<pg, 128, sm, st>>>(d_bnd, deg, coff, ctrl, w, sink, serr, d_order);
  k_prep_deg<4><<<pg, 128, sm, st>>>(d_bnd, deg, coff, ctrl, w, sink, serr, d_order);
  k_prep_deg<3><<<pg, 128, sm, st>>>(d_bnd, deg, coff, ctrl, w, sink, serr, d_order);
  k_prep_deg<2><<<pg, 128, sm, st>>>(d_bnd, deg, coff, ctrl, w, sink, serr, d_order);
  k_prep_deg<1><<<pg, 128, sm, st>>>(d_bnd, deg, coff, ctrl, w, sink, serr, d_order);
  k_prep_bad<<<std::min((n_segs + 255) / 256, 148), 256, 0, st>>>(d_bnd, sink, serr, d_order);
#endif
  g_build_launches += 7;
  return cudaGetLastError();
}

// K2c launch over `ng` device PlanGroups into F's record buffers
template <typename R>
cudaError_t launch_emit(const BuildCtx &B, int ng, const PlanGroup *dg, wn_faces_t F) {
  if (ng <= 0) return cudaSuccess;
  const double rel = (sizeof(R) == 4) ? std::ldexp(1.0, -17) : std::ldexp(1.0, -40);
  ++g_build_launches;
  k_emit<R><<<(int)((32 * (int64_t)ng + 32 * EMIT_WARPS - 1) / (32 * EMIT_WARPS)), 32 * EMIT_WARPS, 0, B.st>>>(
      ng, dg, B.lso, B.loop_face, B.per, B.dom, B.lsta, B.s0, B.inv, B.shift, B.brk, B.chain,
      B.s0pre, B.lend, B.info, (double)rel, (Hot<R> *)F->hot, F->copy, (int32_t)F->n_records, (int32_t)F->n_seg);
  return cudaGetLastError();
}

// emit the records of a HOST `plan` into a new handle whose faces carry
// `fper`/`fdom` (the pairing probes' virtual faces; the main build plans on
// the device)
template <typename R>
wn_status_t materialise(const BuildCtx &B, const Plan &plan, const std::vector<uint8_t> &fper,
                        const std::vector<double> &fdom, const std::vector<double> &fM, void *base_cold,
                        wn_faces_t F) {
  cudaStream_t st = B.st;
  const int nf = (int)fper.size();
  F->n_faces = nf;
  F->n_records = plan.recs;
  F->n_seg = plan.colds;
  F->n_lines = plan.n_lines;
  F->n_groups = plan.n_cull;
  WN_CUDA(cache_alloc((void **)&F->hot, sizeof(Hot<R>) * (size_t)std::max(plan.recs, 1), st));
  F->cold = base_cold;      // the main build's per-segment records (borrowed)
  F->owns_cold = 0;
  WN_CUDA(cache_alloc((void **)&F->copy, sizeof(CopyRec) * (size_t)std::max(plan.colds, 1), st));
  WN_CUDA(cache_alloc((void **)&F->face_rec_off, sizeof(int32_t) * (nf + 1), st));
  WN_CUDA(cache_alloc((void **)&F->face_cold_off, sizeof(int32_t) * (nf + 1), st));
  WN_CUDA(cache_alloc((void **)&F->face_order, sizeof(int32_t) * std::max(nf, 1), st));
  WN_CUDA(cache_alloc((void **)&F->face_dom, sizeof(double) * 4 * std::max(nf, 1), st));
  WN_CUDA(cache_alloc((void **)&F->face_per, std::max(nf, 1), st));
  WN_CUDA(cache_alloc((void **)&F->face_ok, std::max(nf, 1), st));
  WN_CUDA(cache_alloc((void **)&F->face_M, sizeof(double) * std::max(nf, 1), st));
  WN_CUDA(cache_alloc((void **)&F->face_box, sizeof(float4) * std::max(nf, 1), st));
  WN_CUDA(cudaMemsetAsync(F->face_box, 0, sizeof(float4) * std::max(nf, 1), st));   // probes: no regrouping
  WN_CUDA(cache_alloc((void **)&F->counters, 16 * sizeof(unsigned long long), st));
  F->bytes = (int64_t)sizeof(Hot<R>) * plan.recs + (int64_t)sizeof(CopyRec) * plan.colds + (int64_t)nf * 50;
  int32_t maxr = 0;
  for (int f = 0; f < nf; ++f) maxr = std::max(maxr, plan.rec_off[f + 1] - plan.rec_off[f]);
  F->max_face_records = maxr;
  // face_order: faces by decreasing record count, ties by index (stable counting sort)
  static std::vector<int32_t> order, bucket;
  order.resize(nf);
  if ((int64_t)maxr <= 4 * (int64_t)nf + 4096) {
    bucket.assign((size_t)maxr + 2, 0);
    for (int f = 0; f < nf; ++f) ++bucket[maxr - (plan.rec_off[f + 1] - plan.rec_off[f]) + 1];
    for (int32_t c = 0; c <= maxr; ++c) bucket[c + 1] += bucket[c];
    for (int f = 0; f < nf; ++f) order[bucket[maxr - (plan.rec_off[f + 1] - plan.rec_off[f])]++] = f;
  } else {
    std::iota(order.begin(), order.end(), 0);
    std::sort(order.begin(), order.end(), [&](int a, int b) {
      const int ca = plan.rec_off[a + 1] - plan.rec_off[a], cb = plan.rec_off[b + 1] - plan.rec_off[b];
      return ca != cb ? ca > cb : a < b;
    });
  }
  static std::vector<uint8_t> ok;
  ok.assign(nf, 1);
  WN_CUDA(h2d(F->face_rec_off, plan.rec_off.data(), sizeof(int32_t) * (nf + 1), st));
  WN_CUDA(h2d(F->face_cold_off, plan.cold_off.data(), sizeof(int32_t) * (nf + 1), st));
  if (nf) {
    WN_CUDA(h2d(F->face_order, order.data(), sizeof(int32_t) * nf, st));
    WN_CUDA(h2d(F->face_dom, fdom.data(), sizeof(double) * 4 * nf, st));
    WN_CUDA(h2d(F->face_per, fper.data(), nf, st));
    WN_CUDA(h2d(F->face_ok, ok.data(), nf, st));
    WN_CUDA(h2d(F->face_M, fM.data(), sizeof(double) * nf, st));
  }
  const int ng = (int)plan.groups.size();
  if (ng) {
    PlanGroup *dg = nullptr;
    WN_CUDA(cache_alloc((void **)&dg, sizeof(PlanGroup) * ng, st));
    WN_CUDA(h2d(dg, plan.groups.data(), sizeof(PlanGroup) * ng, st));
    WN_CUDA(launch_emit<R>(B, ng, dg, F));
    cache_free(dg, st);
  }
  return WN_OK;
}

}  // namespace

extern "C" wn_status_t wn_build_faces(int32_t n_faces, int32_t n_loops, int32_t n_segs, const double *ctrl_uv,
                                      const double *ctrl_w, const int32_t *seg_degree,
                                      const int32_t *loop_seg_off, const int32_t *face_loop_off,
                                      const uint8_t *face_periodic, const double *face_domain,
                                      const wn_options_t *opts, void *stream, wn_faces_t *out,
                                      int32_t *face_status) {
  set_error("");
  g_build_launches = 0;
  std::lock_guard<std::mutex> build_lock(g_build_mu);
  for (int d = 0; d < 64; ++d)
    if (g_pin_pending[d]) {
      cudaEventSynchronize(g_pin_ev[d]);
      g_pin_pending[d] = false;
    }
  g_pin.reset();
  if (!out) { set_error("wn_build_faces: out == NULL"); return WN_ERR_ARG; }
  if (n_faces < 0 || n_loops < 0 || n_segs < 0) { set_error("wn_build_faces: negative count"); return WN_ERR_ARG; }
  if (!loop_seg_off || !face_loop_off || (n_faces > 0 && (!face_periodic || !face_domain)) ||
      (n_segs > 0 && (!ctrl_uv || !seg_degree))) {
    set_error("wn_build_faces: NULL array");
    return WN_ERR_ARG;
  }
  wn_options_t O;
  O.eps = 0; O.max_depth = 0; O.precision = 0; O.rule = 0; O.angle_mode = 0; O.strict = 1; O.hierarchy = 1;
  if (opts) O = *opts;
  if (O.precision != 0 && O.precision != 1) { set_error("bad precision"); return WN_ERR_ARG; }
  if (O.rule != 0 && O.rule != 1) { set_error("bad rule"); return WN_ERR_ARG; }
  if (O.angle_mode != 0 && O.angle_mode != 1) { set_error("bad angle_mode"); return WN_ERR_ARG; }
  if (O.max_depth < 0 || O.max_depth > 64) { set_error("max_depth must be in [0,64]"); return WN_ERR_ARG; }
  const bool fp32 = O.precision == 1;
  const double eps = O.eps > 0 ? O.eps : (fp32 ? 1e-6 : 1e-10);
  const int maxd = O.max_depth > 0 ? O.max_depth : 48;
  const bool angle = O.angle_mode == 1;
  if (O.hierarchy != 0 && O.hierarchy != 1) { set_error("bad hierarchy option"); return WN_ERR_ARG; }
  int dev = 0;
  {
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  }
  ensure_pool(dev);
  if (dev < 0 || dev >= 64) { set_error("device index out of range"); return WN_ERR_ARG; }
  if (!g_pin_ev[dev]) {
    WN_CUDA(cudaEventCreateWithFlags(&g_pin_ev[dev], cudaEventDisableTiming));
    WN_CUDA(cudaEventCreateWithFlags(&g_ev_lift[dev], cudaEventDisableTiming));
    WN_CUDA(cudaEventCreateWithFlags(&g_ev_plan[dev], cudaEventDisableTiming));
    WN_CUDA(cudaEventCreateWithFlags(&g_ev_fill[dev], cudaEventDisableTiming));
    WN_CUDA(cudaEventCreateWithFlags(&g_ev_k1[dev], cudaEventDisableTiming));
    WN_CUDA(cudaStreamCreateWithFlags(&g_aux[dev], cudaStreamNonBlocking));
  }
  cudaStream_t st = (cudaStream_t)stream;
  PinRelease pin_release{g_pin_ev[dev], &g_pin_pending[dev], st};
  DevBuf D;
  D.st = st;
  Trace tr;

  // --- host copies of the small CSR / face arrays ---
  // (pinned staging: the copies stay asynchronous; read after the plan summary event)
  // (validated on the device, k_csr_check; the pairing path copies what it needs)
  int32_t *h_flo = (int32_t *)g_pin.get(sizeof(int32_t) * (n_faces + 1));
  uint8_t *h_per = (uint8_t *)g_pin.get(std::max(n_faces, 1));
  double *h_dom = (double *)g_pin.get(sizeof(double) * 4 * std::max(n_faces, 1));
  int32_t *h_bad = (int32_t *)g_pin.get(sizeof(int32_t));
  if (!h_flo || !h_per || !h_dom || !h_bad) { set_error("pinned host allocation failed"); return WN_ERR_NOMEM; }
  // --- library copies of the caller's CSR / degree arrays (the caller may free
  // or overwrite every input as soon as this call returns, include/wn.h) ---
  BuildCtx B{};
  B.n_faces = n_faces; B.n_loops = n_loops; B.n_segs = n_segs; B.st = st;
  {
    int32_t *c_deg = nullptr, *c_lso = nullptr, *c_flo = nullptr;
    WN_CUDA(D.alloc(&c_deg, n_segs));
    WN_CUDA(D.alloc(&c_lso, n_loops + 1));
    WN_CUDA(D.alloc(&c_flo, n_faces + 1));
    if (n_segs) WN_CUDA(cudaMemcpyAsync(c_deg, seg_degree, sizeof(int32_t) * n_segs, cudaMemcpyDeviceToDevice, st));
    WN_CUDA(cudaMemcpyAsync(c_lso, loop_seg_off, sizeof(int32_t) * (n_loops + 1), cudaMemcpyDeviceToDevice, st));
    WN_CUDA(cudaMemcpyAsync(c_flo, face_loop_off, sizeof(int32_t) * (n_faces + 1), cudaMemcpyDeviceToDevice, st));
    B.deg = c_deg; B.lso = c_lso; B.flo = c_flo;
  }
  // --- K0: degrees -> control offsets ---
  int32_t *d_cnt = nullptr, *d_bad = nullptr;
  WN_CUDA(D.alloc(&d_cnt, n_segs + 1));
  WN_CUDA(D.alloc(&d_bad, 1));
  WN_CUDA(D.alloc(&B.coff, n_segs + 1));
  WN_CUDA(cudaMemsetAsync(d_bad, 0, sizeof(int32_t), st));
  k_deg<<<(n_segs + 1 + 255) / 256, 256, 0, st>>>(n_segs, B.deg, d_cnt, d_bad);
  g_build_launches += 3;   // k_deg + cub scan (init + scan)
  {
    size_t tmp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp, d_cnt, B.coff, n_segs + 1, st);
    void *dt = nullptr;
    WN_CUDA(D.alloc((char **)&dt, tmp));
    cub::DeviceScan::ExclusiveSum(dt, tmp, d_cnt, B.coff, n_segs + 1, st);
  }
  WN_CUDA(cudaMemcpyAsync(h_bad, d_bad, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  tr.mark("csr copies + degree scan (async)");
  // --- K1 prep, loop->face, K2a lift ---
  uint8_t *d_serr = nullptr;
  WN_CUDA(D.alloc(&B.s0, n_segs));
  WN_CUDA(D.alloc(&d_serr, n_segs));
  WN_CUDA(D.alloc(&B.loop_face, n_loops));
  WN_CUDA(D.alloc(&B.shift, n_segs));
  WN_CUDA(D.alloc(&B.brk, n_segs));
  WN_CUDA(D.alloc(&B.chain, n_segs));
  WN_CUDA(D.alloc(&B.s0pre, n_segs));
  WN_CUDA(D.alloc(&B.lsta, n_segs));
  WN_CUDA(D.alloc(&B.lend, n_segs));
  WN_CUDA(D.alloc(&B.info, n_loops));
  // K2a and K2b (lifting, then the device planner) on an auxiliary stream,
  // concurrent with K1 (derivative bounds: translation invariant, needs no
  // lifting) on `st`; the host waits only for the planner's summary.  Both
  // need the control offsets: the auxiliary stream starts after their scan.
  cudaStream_t st2 = g_aux[dev];
  WN_CUDA(cudaEventRecord(g_ev_lift[dev], st));
  WN_CUDA(cudaStreamWaitEvent(st2, g_ev_lift[dev], 0));
  if (n_loops) WN_CUDA(cudaMemsetAsync(B.loop_face, 0xFF, sizeof(int32_t) * n_loops, st2));
  if (n_faces) k_loop_face<<<(n_faces + 127) / 128, 128, 0, st2>>>(n_faces, n_loops, B.flo, B.loop_face);
  if (n_loops)
    k_lift<<<(int)((32 * (int64_t)n_loops + 255) / 256), 256, 0, st2>>>(n_loops, n_faces, n_segs, B.lso, B.loop_face, face_periodic,
                                                                       face_domain, B.deg, B.coff, ctrl_uv, ctrl_w,
                                                                       B.shift, B.brk, B.chain, B.lsta, B.lend, B.info);
  g_build_launches += (n_faces ? 1 : 0) + (n_loops ? 1 : 0);
  WN_CUDA(cudaGetLastError());
  if (tr.sync) { cudaStreamSynchronize(st2); tr.mark("(trace) k_loop_face + k_lift"); }
  DevBuf D2;
  D2.st = st2;
  wn_faces_t F = new wn_faces_s();
  std::unique_ptr<wn_faces_s, void (*)(wn_faces_s *)> F_guard(F, [](wn_faces_s *p) { free_handle(p); });
  F->precision = fp32 ? 1 : 0;
  F->opt = O;
  F->eps = eps;
  F->max_depth = maxd;
  F->device = dev;
  F->n_faces = n_faces;
  const int nf1 = std::max(n_faces, 1);
  WN_CUDA(cache_alloc((void **)&F->face_rec_off, sizeof(int32_t) * (n_faces + 1), st2));
  WN_CUDA(cache_alloc((void **)&F->face_cold_off, sizeof(int32_t) * (n_faces + 1), st2));
  WN_CUDA(cache_alloc((void **)&F->face_order, sizeof(int32_t) * nf1, st2));
  WN_CUDA(cache_alloc((void **)&F->face_dom, sizeof(double) * 4 * nf1, st2));
  WN_CUDA(cache_alloc((void **)&F->face_per, nf1, st2));
  WN_CUDA(cache_alloc((void **)&F->face_ok, nf1, st2));
  WN_CUDA(cache_alloc((void **)&F->face_M, sizeof(double) * nf1, st2));
  WN_CUDA(cache_alloc((void **)&F->face_box, sizeof(float4) * nf1, st2));
  WN_CUDA(cache_alloc((void **)&F->counters, 16 * sizeof(unsigned long long), st2));
  // the emission reads the handle's face arrays (written by k_plan_count:
  // periodicity bits, domain with non-periodic axes zeroed) -- library-owned
  B.per = F->face_per;
  B.dom = F->face_dom;
  int32_t *d_status = face_status;
  if (!d_status) WN_CUDA(D2.alloc(&d_status, nf1));
  int4 *d_cnt4 = nullptr, *d_off4 = nullptr;
  uint32_t *d_okey = nullptr, *d_okey2 = nullptr;
  int32_t *d_oval = nullptr;
  BuildSummary *d_sum = nullptr;
  WN_CUDA(D2.alloc(&d_cnt4, nf1));
  WN_CUDA(D2.alloc(&d_off4, nf1));
  WN_CUDA(D2.alloc(&d_okey, nf1));
  WN_CUDA(D2.alloc(&d_okey2, nf1));
  WN_CUDA(D2.alloc(&d_oval, nf1));
  WN_CUDA(D2.alloc(&d_sum, 1));
  size_t sort_tmp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, sort_tmp, d_okey, d_okey2, d_oval, F->face_order, n_faces, 0, 32, st2);
  char *d_sort_tmp = nullptr;
  WN_CUDA(D2.alloc(&d_sort_tmp, std::max(sort_tmp, (size_t)16)));
  BuildSummary *h_sum = (BuildSummary *)g_pin.get(sizeof(BuildSummary));
  if (!h_sum) { set_error("pinned host allocation failed"); return WN_ERR_NOMEM; }
  if (n_faces) WN_CUDA(cudaMemsetAsync(F->face_ok, 1, n_faces, st2));

  auto plan_pass = [&](const int *pair_beta, const int *pair_s) -> wn_status_t {
    WN_CUDA(cudaMemsetAsync(d_sum, 0, sizeof(BuildSummary), st2));
    WN_CUDA(cudaMemsetAsync(&d_sum->first_bad, 0xFF, sizeof(unsigned long long), st2));
    WN_CUDA(cudaMemsetAsync(&d_sum->dom_bad, 0xFF, sizeof(unsigned), st2));
    if (!pair_beta) {
      k_csr_check<<<(std::max(n_loops, n_faces) + 1 + 255) / 256, 256, 0, st2>>>(n_loops, n_faces, n_segs, B.lso, B.flo,
                                                                                face_periodic, face_domain, d_sum);
      ++g_build_launches;
    }
    if (n_faces) {
      k_plan_count<<<(n_faces + 127) / 128, 128, 0, st2>>>(
          n_faces, n_loops, B.flo, face_periodic, face_domain, B.info, angle ? 1 : 0, O.strict ? 1 : 0,
          O.hierarchy ? 1 : 0, fp32 ? 1 : 0, pair_beta, pair_s, d_status, F->face_per, F->face_dom, F->face_M,
          F->face_box, d_cnt4, d_okey, d_oval, d_sum);
      k_plan_scan<<<1, PLAN_SCAN_T, 0, st2>>>(n_faces, d_cnt4, d_off4, F->face_rec_off, F->face_cold_off, d_sum);
      WN_CUDA(cub::DeviceRadixSort::SortPairs(d_sort_tmp, sort_tmp, d_okey, d_okey2, d_oval, F->face_order, n_faces,
                                              0, 32, st2));
      g_build_launches += 2 + 4;
    } else {
      WN_CUDA(cudaMemsetAsync(F->face_rec_off, 0, sizeof(int32_t), st2));
      WN_CUDA(cudaMemsetAsync(F->face_cold_off, 0, sizeof(int32_t), st2));
    }
    WN_CUDA(cudaGetLastError());
    WN_CUDA(cudaMemcpyAsync(h_sum, d_sum, sizeof(BuildSummary), cudaMemcpyDeviceToHost, st2));
    WN_CUDA(cudaEventRecord(g_ev_plan[dev], st2));
    return WN_OK;
  };
  {
    wn_status_t rc = plan_pass(nullptr, nullptr);
    if (rc != WN_OK) return rc;
  }
  // K1 (reads the caller's control points: the host waits for g_ev_k1 before returning)
  // K1 writes the handle's per-segment cold records (BaseCold) and S0
  F->n_base = n_segs;
  WN_CUDA(cache_alloc((void **)&F->inv, sizeof(int32_t) * (size_t)std::max(n_segs, 1), st));
  B.inv = F->inv;
  WN_CUDA(cache_alloc(&F->cold, (fp32 ? sizeof(BaseCold<float>) : sizeof(BaseCold<double>)) * (size_t)std::max(n_segs, 1),
                      st));
  if (fp32)
    WN_CUDA(launch_k1(n_segs, B.deg, B.coff, ctrl_uv, ctrl_w,
                      ColdSink<float>{(BaseCold<float> *)F->cold, B.s0, F->inv, std::ldexp(1.0, -17)}, d_serr, D, st));
  else
    WN_CUDA(launch_k1(n_segs, B.deg, B.coff, ctrl_uv, ctrl_w,
                      ColdSink<double>{(BaseCold<double> *)F->cold, B.s0, F->inv, std::ldexp(1.0, -40)}, d_serr, D, st));
  if (n_loops) {
    k_s0pre<<<(int)((32 * (int64_t)n_loops + 255) / 256), 256, 0, st>>>(n_loops, n_segs, B.lso, B.s0, B.s0pre);
    ++g_build_launches;
  }
  WN_CUDA(cudaGetLastError());
  WN_CUDA(cudaEventRecord(g_ev_k1[dev], st));
  if (tr.sync) { cudaStreamSynchronize(st); tr.mark("(trace) k_prep + k_s0pre"); }
  WN_CUDA(cudaEventSynchronize(g_ev_plan[dev]));
  tr.mark("device plan summary");
  // CSR / domain checks on the host (the kernels above clamp every CSR index,
  // so a bad input is reported here without any out-of-bounds access).  An
  // error return also waits for K1 (it reads the caller's arrays).
  auto fail = [&](wn_status_t rc) {
    cudaStreamSynchronize(st2);
    cudaEventSynchronize(g_ev_k1[dev]);
    return rc;
  };
  if (h_sum->csr_bad) { set_error("wn_build_faces: bad loop/face CSR offsets"); return fail(WN_ERR_ARG); }
  if (*h_bad) { set_error("wn_build_faces: segment degree outside 1..5"); return fail(WN_ERR_ARG); }
  if (h_sum->dom_bad != 0xFFFFFFFFu) {
    set_error("face %u: bad %s period", h_sum->dom_bad >> 1, (h_sum->dom_bad & 1) ? "v" : "u");
    return fail(WN_ERR_GEOM);
  }
  auto report_bad = [&]() {
    const int first = (int)(h_sum->first_bad >> 32), code = (int)(h_sum->first_bad & 0xffffffffu);
    set_error("wn_build_faces: face %d invalid (code %d)", first, code);
    return fail(h_sum->geom ? WN_ERR_GEOM : (h_sum->unsup ? WN_ERR_UNSUPPORTED : WN_ERR_TOPOLOGY));
  };
  if (h_sum->bad) return report_bad();
  tr.mark("host checks");

  const int *d_pair_beta = nullptr, *d_pair_s = nullptr;
  if (h_sum->needp) {
    // --- pairing (Algs. 7-9) for bi-periodic faces via probe queries (host) ---
    WN_CUDA(cudaMemcpyAsync(h_flo, B.flo, sizeof(int32_t) * (n_faces + 1), cudaMemcpyDeviceToHost, st2));
    if (n_faces) {
      WN_CUDA(cudaMemcpyAsync(h_per, face_periodic, n_faces, cudaMemcpyDeviceToHost, st2));
      WN_CUDA(cudaMemcpyAsync(h_dom, face_domain, sizeof(double) * 4 * n_faces, cudaMemcpyDeviceToHost, st2));
    }
    LoopInfo *L = (LoopInfo *)g_pin.get(sizeof(LoopInfo) * std::max(n_loops, 1));
    if (!L) { set_error("pinned host allocation failed"); return fail(WN_ERR_NOMEM); }
    if (n_loops) WN_CUDA(cudaMemcpyAsync(L, B.info, sizeof(LoopInfo) * n_loops, cudaMemcpyDeviceToHost, st2));
    WN_CUDA(cudaStreamSynchronize(st2));
    std::vector<FaceCtx> ctx(n_faces);
    std::vector<int32_t> status(n_faces, WN_FACE_OK);
    std::vector<int> need_pair;
    for (int f = 0; f < n_faces; ++f) {
      ctx[f] = face_ctx(h_per[f], &h_dom[4 * f], angle);
      ctx[f].M = face_margin(L, h_flo[f], h_flo[f + 1], ctx[f], fp32);
      int np = 0;
      face_validate(L, h_flo[f], h_flo[f + 1], ctx[f], O.strict != 0, &np);
      if (np) need_pair.push_back(f);
    }
    // Candidates (R16): the beta-translates modulo alpha's extension vector,
    // indexed by the band offset s (axis classes: the transverse lattice
    // index; general classes (p,q): m = p*j - q*i, with the translate moved
    // along v next to alpha so the probe stays near the emitted copies).
    struct Cand { int face, alpha, beta, s, ti, tj; double px, py; };
    std::vector<int> pair_beta(n_loops, -1), pair_s(n_loops, 0);
    std::vector<Cand> cands;
    auto face_class = [&](int f, int &cp, int &cq) {
      cp = cq = 0;
      for (int l = h_flo[f]; l < h_flo[f + 1]; ++l)
        if (L[l].nseg && (L[l].cu || L[l].cv)) { cp = L[l].cu; cq = L[l].cv; break; }
    };
    for (int f : need_pair) {
      const FaceCtx &C = ctx[f];
      int cp, cq;
      face_class(f, cp, cq);
      const bool general = cp != 0 && cq != 0;
      const int tax = (cp != 0) ? 1 : 0;                // transverse axis (axis classes)
      const double Tt = tax ? C.Tv : C.Tu;
      const double vx = cp * C.Tu, vy = cq * C.Tv;
      for (int la = h_flo[f]; la < h_flo[f + 1]; ++la) {
        if (!(L[la].nseg && L[la].cu == cp && L[la].cv == cq)) continue;
        for (int lb = h_flo[f]; lb < h_flo[f + 1]; ++lb) {
          if (!(L[lb].nseg && L[lb].cu == -cp && L[lb].cv == -cq)) continue;
          int J;
          if (general) {
            double alo, ahi, blo, bhi;
            box_nu(L[la].bb, cp, cq, C, 0, 0, alo, ahi);
            box_nu(L[lb].bb, cp, cq, C, 0, 0, blo, bhi);
            J = 3 + (int)std::ceil((bhi - blo) + std::fabs(alo - blo));
          } else {
            const double ext = tax ? (L[lb].bb[3] - L[lb].bb[1]) / Tt : (L[lb].bb[2] - L[lb].bb[0]) / Tt;
            const double da = tax ? (L[la].bb[1] - L[lb].bb[1]) / Tt : (L[la].bb[0] - L[lb].bb[0]) / Tt;
            J = 3 + (int)std::ceil(ext + std::fabs(da));
          }
          for (int sidx = -J; sidx <= J; ++sidx) {
            int ti = tax ? 0 : sidx, tj = tax ? sidx : 0;
            if (general) {
              band_rep(cp, cq, sidx, ti, tj);
              const double dx = L[la].sx - (L[lb].sx + ti * C.Tu), dy = L[la].sy - (L[lb].sy + tj * C.Tv);
              const int k = (int)std::lround((dx * vx + dy * vy) / (vx * vx + vy * vy));
              ti += k * cp;
              tj += k * cq;
            }
            cands.push_back({f, la, lb, sidx, ti, tj, L[lb].sx + ti * C.Tu, L[lb].sy + tj * C.Tv});
          }
        }
      }
    }
    // virtual faces: one extended curve per non-contractible loop.  Axis
    // classes: a uni-periodic face along the class axis (queries reduced along
    // it).  General classes: a face without reduction (per = 4) holding the
    // slanted line and every copy that can contain a probe point.
    std::vector<int> vface(n_loops, -1);
    std::vector<double> tmin(n_loops, INFINITY), tmax(n_loops, -INFINITY);
    auto cover = [&](int l, double x, double y, const FaceCtx &C) {
      const double vx = L[l].cu * C.Tu, vy = L[l].cv * C.Tv;
      const double t = ((x - L[l].sx) * vx + (y - L[l].sy) * vy) / (vx * vx + vy * vy);
      tmin[l] = std::min(tmin[l], t);
      tmax[l] = std::max(tmax[l], t);
    };
    for (size_t i = 0; i < cands.size(); ++i) {
      const Cand &a = cands[i];
      const FaceCtx &C = ctx[a.face];
      if (!(L[a.alpha].cu && L[a.alpha].cv)) continue;
      cover(a.alpha, a.px, a.py, C);                    // batch 1: omega(pt(beta~), alpha_ext)
      for (size_t j = 0; j < cands.size(); ++j)         // batch 2 (any later left pair)
        if (j != i && cands[j].alpha == a.alpha)
          cover(cands[j].beta, a.px - cands[j].ti * C.Tu, a.py - cands[j].tj * C.Tv, C);
    }
    Plan VP;
    std::vector<uint8_t> vper;
    std::vector<double> vdom, vM;
    for (int f : need_pair) {
      for (int l = h_flo[f]; l < h_flo[f + 1]; ++l) {
        const LoopInfo &I = L[l];
        if (I.nseg == 0 || (I.cu == 0 && I.cv == 0)) continue;
        FaceCtx C = ctx[f];
        C.angle = false;
        const bool general = I.cu != 0 && I.cv != 0;
        const int axis = (I.cu != 0) ? 0 : 1;
        vface[l] = (int)vper.size();
        vper.push_back(general ? 4 : (axis == 0 ? 1 : 2));
        vdom.insert(vdom.end(), {ctx[f].u0, ctx[f].Tu, ctx[f].v0, ctx[f].Tv});
        vM.push_back(C.M);
        VP.begin_face(vface[l]);
        VP.add(G_LINE, 0, l, 0, 0, I, C.M);
        if (!general) {
          C.per = axis == 0 ? 1 : 2;
          plan_extended_copies(VP, l, I, C, axis, 0, false, O.hierarchy != 0);
        } else if (tmin[l] <= tmax[l]) {
          const double vx = I.cu * C.Tu, vy = I.cv * C.Tv;
          const double E = 2.0 * std::hypot(I.bb[2] - I.bb[0], I.bb[3] - I.bb[1]) / std::hypot(vx, vy) + 1.0;
          const int k0 = (int)std::floor(tmin[l] - E) - 1, k1 = (int)std::ceil(tmax[l] + E) + 1;
          const int fl = loop_flags(I, false, true, O.hierarchy != 0);
          for (int k = k0; k <= k1; ++k) VP.add(G_COPY, fl, l, k * I.cu, k * I.cv, I, C.M);
        }
      }
    }
    VP.end();
    struct QueryRec { int vf; double x, y; };
    std::vector<QueryRec> qs;
    for (const Cand &c : cands) qs.push_back({vface[c.alpha], c.px, c.py});
    // run probes through the query kernel on a temporary handle (fp64, crossing mode)
    // the probes run fp64 records: an fp32 build gets fp64 base cold records for them
    void *probe_cold = F->cold;
    if (fp32) {
      double *tmp_s0 = nullptr;
      WN_CUDA(D.alloc((BaseCold<double> **)&probe_cold, std::max(n_segs, 1)));
      WN_CUDA(D.alloc(&tmp_s0, std::max(n_segs, 1)));
      WN_CUDA(launch_k1(n_segs, B.deg, B.coff, ctrl_uv, ctrl_w,
                        ColdSink<double>{(BaseCold<double> *)probe_cold, tmp_s0, F->inv, std::ldexp(1.0, -40)}, d_serr, D,
                        st));
    }
    WN_CUDA(cudaStreamSynchronize(st));   // K1 outputs (bounds, span prefixes) are read by the probes' k_emit
    auto run_probes = [&](const std::vector<QueryRec> &Q, std::vector<double> &res) -> wn_status_t {
      wn_faces_t T = new wn_faces_s();
      T->precision = 0; T->eps = 1e-12; T->max_depth = 60; T->device = dev; T->opt = O; T->opt.rule = 0; T->opt.angle_mode = 0;   // the probe records are crossing-mode (C.angle = false)
      wn_status_t rc = materialise<double>(B, VP, vper, vdom, vM, probe_cold, T);
      T->n_base = n_segs;
      if (rc != WN_OK) { free_handle(T); return rc; }
      const int nq = (int)Q.size();
      std::vector<int32_t> hf(nq);
      std::vector<double> huv(2 * (size_t)nq);
      for (int i = 0; i < nq; ++i) { hf[i] = Q[i].vf; huv[2 * i] = Q[i].x; huv[2 * i + 1] = Q[i].y; }
      int32_t *df = nullptr; double *duv = nullptr, *dw = nullptr; uint8_t *dfl = nullptr;
      DevBuf Q2; Q2.st = st;
      WN_CUDA(Q2.alloc(&df, nq)); WN_CUDA(Q2.alloc(&duv, 2 * (size_t)nq));
      WN_CUDA(Q2.alloc(&dw, nq)); WN_CUDA(Q2.alloc(&dfl, nq));
      WN_CUDA(cudaMemcpyAsync(df, hf.data(), sizeof(int32_t) * nq, cudaMemcpyHostToDevice, st));
      WN_CUDA(cudaMemcpyAsync(duv, huv.data(), sizeof(double) * 2 * nq, cudaMemcpyHostToDevice, st));
      rc = wn_query(T, nq, df, duv, dw, dfl, st);
      g_build_launches += wn_last_query_launches();
      res.resize(nq);
      if (rc == WN_OK) {
        WN_CUDA(cudaMemcpyAsync(res.data(), dw, sizeof(double) * nq, cudaMemcpyDeviceToHost, st));
        WN_CUDA(cudaStreamSynchronize(st));
      }
      free_handle(T);
      return rc;
    };
    std::vector<double> r1;
    wn_status_t rc = run_probes(qs, r1);
    if (rc != WN_OK) return fail(rc);
    // candidates left of alpha (ToLeft, Alg. 7: omega > 0)
    std::vector<int> left;
    for (size_t i = 0; i < cands.size(); ++i)
      if (r1[i] > 0.0) left.push_back((int)i);
    // pairwise ToLeft(c1, c2) among left candidates of the same alpha
    std::vector<QueryRec> q2;
    std::vector<std::pair<int, int>> q2pairs;
    for (int i : left)
      for (int j : left) {
        if (i == j || cands[i].alpha != cands[j].alpha) continue;
        const Cand &a = cands[i], &bb = cands[j];
        const FaceCtx &C = ctx[a.face];
        // omega(pt(c1) - t2, beta2_ext) (translation identity, App. C.1)
        q2.push_back({vface[bb.beta], a.px - bb.ti * C.Tu, a.py - bb.tj * C.Tv});
        q2pairs.push_back({i, j});
      }
    std::vector<double> r2;
    if (!q2.empty()) {
      rc = run_probes(q2, r2);
      if (rc != WN_OK) return fail(rc);
    }
    auto to_left = [&](int i, int j) {
      for (size_t k = 0; k < q2pairs.size(); ++k)
        if (q2pairs[k].first == i && q2pairs[k].second == j) return r2[k] > 0.0;
      return false;
    };
    // Alg. 9 PairLoops: greedy nearest-left proper translate per alpha
    std::vector<uint8_t> used(n_loops, 0);
    int pairing_failed = -1;
    for (int f : need_pair) {
      for (int la = h_flo[f]; la < h_flo[f + 1]; ++la) {
        bool is_alpha = false;
        for (int i : left) if (cands[i].alpha == la) { is_alpha = true; break; }
        const LoopInfo &Ia = L[la];
        int cp = 0, cq = 0;
        for (int l = h_flo[f]; l < h_flo[f + 1]; ++l)
          if (L[l].nseg && (L[l].cu || L[l].cv)) { cp = L[l].cu; cq = L[l].cv; break; }
        if (!(Ia.nseg && Ia.cu == cp && Ia.cv == cq)) continue;
        int best = -1;
        if (is_alpha)
          for (int i : left) {
            if (cands[i].alpha != la || used[cands[i].beta]) continue;
            if (best < 0 || to_left(i, best)) best = i;
          }
        if (best < 0) { status[f] = WN_FACE_PAIRING; if (pairing_failed < 0) pairing_failed = f; break; }
        used[cands[best].beta] = 1;
        pair_beta[la] = cands[best].beta;
        pair_s[la] = cands[best].s;
      }
    }
    if (pairing_failed >= 0) {
      if (face_status) {
        for (int f = 0; f < n_faces; ++f)
          if (status[f]) WN_CUDA(cudaMemcpyAsync(face_status + f, &status[f], sizeof(int32_t), cudaMemcpyHostToDevice, st2));
      }
      set_error("wn_build_faces: face %d invalid (code %d)", pairing_failed, (int)WN_FACE_PAIRING);
      return fail(WN_ERR_TOPOLOGY);
    }
    int *d_pb = nullptr, *d_ps = nullptr;
    WN_CUDA(D2.alloc(&d_pb, std::max(n_loops, 1)));
    WN_CUDA(D2.alloc(&d_ps, std::max(n_loops, 1)));
    if (n_loops) {
      WN_CUDA(h2d(d_pb, pair_beta.data(), sizeof(int) * n_loops, st2));
      WN_CUDA(h2d(d_ps, pair_s.data(), sizeof(int) * n_loops, st2));
    }
    rc = plan_pass(d_pb, d_ps);
    if (rc != WN_OK) return fail(rc);
    WN_CUDA(cudaEventSynchronize(g_ev_plan[dev]));
    if (h_sum->bad) return report_bad();
    tr.mark("pairing probes + re-plan");
    // the fill pass below also needs the pairs
    d_pair_beta = d_pb;
    d_pair_s = d_ps;
  }
  if (h_sum->toobig) { set_error("too many records (22/24-bit record indices)"); return fail(WN_ERR_ARG); }

  // --- K2c: record buffers, group fill (aux stream), emission (after K1) ---
  F->n_records = h_sum->tot_r;
  F->n_seg = h_sum->tot_c;
  F->n_lines = (int64_t)h_sum->lines;
  F->n_groups = (int64_t)h_sum->cull;
  F->n_copy_groups = (int64_t)h_sum->copies;
  F->n_bands = (int64_t)h_sum->bands;
  F->max_face_records = h_sum->maxr;
  WN_CUDA(cache_alloc(&F->hot, (fp32 ? sizeof(Hot<float>) : sizeof(Hot<double>)) * (size_t)std::max(h_sum->tot_r, 1), st));
  WN_CUDA(cache_alloc((void **)&F->copy, sizeof(CopyRec) * (size_t)std::max(h_sum->tot_c, 1), st));
  F->bytes = (int64_t)(fp32 ? sizeof(Hot<float>) : sizeof(Hot<double>)) * h_sum->tot_r +
             (int64_t)(fp32 ? sizeof(BaseCold<float>) : sizeof(BaseCold<double>)) * n_segs +
             (int64_t)sizeof(CopyRec) * h_sum->tot_c + (int64_t)n_faces * 50;
  const int ng = h_sum->tot_g;
  // the plan groups: written by k_plan_fill on st2, read by k_emit on st --
  // released on st (after k_emit), not with the auxiliary stream's buffers
  PlanGroup *d_groups = nullptr;
  WN_CUDA(cache_alloc((void **)&d_groups, sizeof(PlanGroup) * (size_t)std::max(ng, 1), st2));
  struct GroupsRelease {
    void *p;
    cudaStream_t st;
    ~GroupsRelease() { cache_free(p, st); }
  } groups_release{d_groups, st};
  if (ng) {
    k_plan_fill<<<(n_faces + 127) / 128, 128, 0, st2>>>(n_faces, n_loops, B.flo, F->face_per, F->face_dom,
                                                        F->face_M, B.info, angle ? 1 : 0, O.hierarchy ? 1 : 0,
                                                        d_pair_beta, d_pair_s, d_off4, d_groups);
    ++g_build_launches;
    WN_CUDA(cudaGetLastError());
  }
  WN_CUDA(cudaEventRecord(g_ev_fill[dev], st2));
  WN_CUDA(cudaStreamWaitEvent(st, g_ev_fill[dev], 0));   // join: K2c after the plan and after K1
  WN_CUDA(fp32 ? launch_emit<float>(B, ng, d_groups, F) : launch_emit<double>(B, ng, d_groups, F));
  tr.mark("device plan fill + emit (enqueued)");
  // K1 is the last reader of the caller's buffers (k_emit reads the library's
  // lifted copies): once it is done the inputs may be freed (include/wn.h).
  // The emission is already queued behind it, so this wait leaves no gap.
  WN_CUDA(cudaEventSynchronize(g_ev_k1[dev]));
  tr.mark("K1 done (inputs released)");
  // no final synchronisation: the handle's records are complete in stream
  // order, so queries enqueued on `stream` after this call see them
  {
    cudaError_t e = cudaEventCreateWithFlags(&F->last_use, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&F->ready, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventRecord(F->last_use, st);
    if (e == cudaSuccess) e = cudaEventRecord(F->ready, st);
    if (e != cudaSuccess) return cuda_fail(e, "build event");
  }
  if (tr.sync) { cudaStreamSynchronize(st); tr.mark("(trace) k_plan_fill + k_emit"); }
  *out = F_guard.release();
  return WN_OK;
}

extern "C" wn_status_t wn_segment_prep(int32_t n_segs, const double *ctrl_uv, const double *ctrl_w,
                                       const int32_t *seg_degree, double *out, void *stream) {
  set_error("");
  if (n_segs < 0 || (n_segs > 0 && (!ctrl_uv || !seg_degree || !out))) {
    set_error("wn_segment_prep: bad arguments");
    return WN_ERR_ARG;
  }
  if (n_segs == 0) return WN_OK;
  std::lock_guard<std::mutex> build_lock(g_build_mu);   // K1's side streams / events are shared with builds
  int dev = 0;
  WN_CUDA(cudaGetDevice(&dev));
  ensure_pool(dev);
  cudaStream_t st = (cudaStream_t)stream;
  DevBuf D;
  D.st = st;
  int32_t *cnt = nullptr, *bad = nullptr, *coff = nullptr;
  uint8_t *serr = nullptr;
  WN_CUDA(D.alloc(&cnt, n_segs + 1));
  WN_CUDA(D.alloc(&bad, 1));
  WN_CUDA(D.alloc(&coff, n_segs + 1));
  WN_CUDA(D.alloc(&serr, n_segs));
  WN_CUDA(cudaMemsetAsync(bad, 0, sizeof(int32_t), st));
  k_deg<<<(n_segs + 1 + 255) / 256, 256, 0, st>>>(n_segs, seg_degree, cnt, bad);
  size_t tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt, coff, n_segs + 1, st);
  char *dt = nullptr;
  WN_CUDA(D.alloc(&dt, tmp));
  cub::DeviceScan::ExclusiveSum(dt, tmp, cnt, coff, n_segs + 1, st);
  int32_t h_bad = 0;
  WN_CUDA(cudaMemcpyAsync(&h_bad, bad, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  WN_CUDA(cudaStreamSynchronize(st));
  if (h_bad) { set_error("wn_segment_prep: segment degree outside 1..5"); return WN_ERR_ARG; }
  // K1 writes 16-B vectors: stage through an aligned buffer if needed.  The
  // same launch sequence as wn_build_faces (launch_k1), so the bound tests
  // through this entry point cover the shipped K1 code.
  SegPrep *dst = (SegPrep *)out;
  if ((uintptr_t)out & 15) WN_CUDA(D.alloc(&dst, n_segs));
  WN_CUDA(launch_k1(n_segs, seg_degree, coff, ctrl_uv, ctrl_w, PrepSink{dst}, serr, D, st));
  if ((void *)dst != (void *)out)
    WN_CUDA(cudaMemcpyAsync(out, dst, sizeof(SegPrep) * (size_t)n_segs, cudaMemcpyDeviceToDevice, st));
  WN_CUDA(cudaGetLastError());
  WN_CUDA(cudaStreamSynchronize(st));
  return WN_OK;
}

namespace wn {
namespace {
template <typename R>
__global__ void k_rec_bounds(int32_t n, const BaseCold<R> *__restrict__ C, const int32_t *__restrict__ inv,
                             double *__restrict__ out) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const BaseCold<R> &c = C[inv[s]];
  double *o = out + 23 * (size_t)s;
  o[0] = (double)c.B;
  for (int q = 0; q < 8; ++q) o[1 + q] = (double)c.Bq[q];
  for (int i = 0; i < 14; ++i) o[9 + i] = (double)c.Sp[i];
}
}  // namespace
}  // namespace wn

extern "C" wn_status_t wn_recursion_bounds(wn_faces_t F, double *out, void *stream) {
  if (!F || (!out && F->n_base > 0)) { set_error("wn_recursion_bounds: NULL"); return WN_ERR_ARG; }
  if (F->n_base == 0) return WN_OK;
  cudaStream_t st = (cudaStream_t)stream;
  WN_CUDA(cudaSetDevice(F->device));
  if (F->ready) WN_CUDA(cudaStreamWaitEvent(st, F->ready, 0));
  const int n = F->n_base;
  if (F->precision == 1)
    k_rec_bounds<float><<<(n + 255) / 256, 256, 0, st>>>(n, (const BaseCold<float> *)F->cold, F->inv, out);
  else
    k_rec_bounds<double><<<(n + 255) / 256, 256, 0, st>>>(n, (const BaseCold<double> *)F->cold, F->inv, out);
  WN_CUDA(cudaGetLastError());
  WN_CUDA(cudaStreamSynchronize(st));
  return WN_OK;
}

extern "C" wn_status_t wn_faces_info(wn_faces_t F, wn_faces_info_t *out) {
  if (!F || !out) { set_error("wn_faces_info: NULL"); return WN_ERR_ARG; }
  out->n_records = F->n_records;
  out->n_seg_records = F->n_seg;
  out->n_groups = F->n_groups;
  out->n_lines = F->n_lines;
  out->bytes = F->bytes;
  out->precision = F->precision;
  out->max_face_records = F->max_face_records;
  out->n_copy_groups = F->n_copy_groups;
  out->n_bands = F->n_bands;
  return WN_OK;
}

extern "C" wn_status_t wn_set_counters(wn_faces_t F, int enable) {
  if (!F) { set_error("wn_set_counters: NULL"); return WN_ERR_ARG; }
  F->counters_on = enable ? 1 : 0;
  return WN_OK;
}

extern "C" wn_status_t wn_get_counters(wn_faces_t F, void *stream, int64_t *out) {
  if (!F || !out) { set_error("wn_get_counters: NULL"); return WN_ERR_ARG; }
  unsigned long long h[12];
  WN_CUDA(cudaMemcpyAsync(h, F->counters, sizeof(h), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  WN_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  for (int i = 0; i < 12; ++i) out[i] = (int64_t)h[i];
  return WN_OK;
}

extern "C" void wn_free_faces(wn_faces_t F) { free_handle(F); }

extern "C" const char *wn_last_error(void) { return wn::g_err; }

extern "C" int32_t wn_last_build_launches(void) { return wn::g_build_launches; }
