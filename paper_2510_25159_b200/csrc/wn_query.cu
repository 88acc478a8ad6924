// wn_query.cu -- the hot path of libwn: query bucketing (K4) and the query
// kernel (K3).  PAPER.md is cited as P:<line>; SURVEY.md rows as 8(a)a3..a8.
//
// K3 maps one query to one thread and one tile of <= 256 queries of a single
// face to one CTA.  The face's hot record program is staged in shared memory
// with 1-D TMA bulk copies (cp.async.bulk + mbarrier) and swept by every warp
// in lock-step, so each record is a broadcast shared-memory read reused by all
// queries of the tile.  Phase 1 (a4/a5/a7) evaluates the root ellipse test of
// Alg. 1 for every (query, segment) pair and substitutes the chord
// of every pruned segment; pairs whose ellipse contains the query ("hard",
// a6) are appended to per-warp shared-memory queues.  Phase 2 drains all the
// CTA's queues with dynamic work fetching: each lane runs Alg. 1's recursion
// (midpoint split, Eq. 2 sub-span bound, P:305-322 / P:351-356) with an
// explicit stack.  a8 reduces, classifies and stores.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <type_traits>

#include "wn_common.cuh"

namespace wn {

// ---------------------------------------------------------------------------
// PTX helpers: 1-D TMA bulk copy global -> shared completed on an mbarrier
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void *p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, "
      "p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// Reduce a periodic coordinate into [x0, x0+T); bit-exact when already inside
// (SURVEY 8(a) a7).  Explicit _rn ops: no FMA contraction, same roundings as
// the definition (the oracle uses the same formula).
__device__ __forceinline__ double reduce_coord(double x, double x0, double T) {
  if (x >= x0 && x < __dadd_rn(x0, T)) return x;
  double d = __dsub_rn(x, x0);
  double r = __dadd_rn(x0, __dsub_rn(d, __dmul_rn(T, floor(__ddiv_rn(d, T)))));
  if (r >= __dadd_rn(x0, T)) r = x0;
  return r;
}

template <typename R>
struct QParams {
  const Hot<R> *hot;
  const BaseCold<R> *cold;   // per input segment
  const CopyRec *copy;       // per emitted segment
  int64_t nq;                // queries of the batch (checked build: index bounds)
  int32_t n_copy, n_base, n_rec;
  const int32_t *face_rec_off;
  const int32_t *face_cold_off;
  const double *face_dom;
  const uint8_t *face_per;
  const double *face_M;
  const double *uv;
  double *winding;
  uint8_t *flag;
  const Tile *tiles;
  const int32_t *ntiles;
  const int32_t *perm;
  const int32_t *unsorted;
  HardEntry *hq;          // global hard-pair queue
  int32_t *hq_count;
  int32_t *hq_next;       // k_hard's dynamic fetch cursor (zeroed with the flags)
  int32_t hq_cap;
  double eps;
  int max_depth;
  int rule;
  unsigned long long *counters;
  // implicit-grid batches (wn_query_grid; grid_box == nullptr: explicit uv):
  // query q = g * grid_n + iv * grid_nu + iu is the cell centre (iu, iv) of
  // grid g over the box grid_box[g] = (u_lo, v_lo, u_hi, v_hi) of face grid_face[g]
  const double2 *grid_box;  // [n_grid][2] = (u_lo, v_lo), (u_hi, v_hi)
  const int32_t *grid_face;
  int64_t grid_n;
  int32_t grid_nu, grid_nv;
  int32_t grid_blk;        // > 0: warp = grid_blk x (32 / grid_blk) cell block (see k_phase1)
  const float4 *face_box;  // [n_faces] box of the face's queries that can be inside (spatial regrouping)
  int32_t spatial;         // explicit batches: regroup each unit's queries in Morton order
  int32_t *sorder;         // [n] regrouped query order, unit by unit (positions of the tile ranges)
  int32_t *skey;           // [n] scratch of the regrouping (cell key << 12 | rank in cell)
};

// Cell-centred grid point (iu + 1/2) * (hi - lo) / n + lo, rounded step by step
// in exactly this order (no contraction): the uv an explicit batch built by
// lo + (i + 0.5) * ((hi - lo) / n) carries, bit for bit.
__device__ __forceinline__ double grid_coord(double lo, double hi, int i, int n) {
  return __dadd_rn(lo, __dmul_rn((double)i + 0.5, __ddiv_rn(__dsub_rn(hi, lo), (double)n)));
}
template <typename R>
__device__ __forceinline__ void grid_point(const QParams<R> &P, int64_t q, double &u, double &v) {
  const int64_t g = q / P.grid_n;
  const int loc = (int)(q - g * P.grid_n);
  const int iv = loc / P.grid_nu, iu = loc - iv * P.grid_nu;
  const double2 lo = __ldg(P.grid_box + 2 * g), hi = __ldg(P.grid_box + 2 * g + 1);
  u = grid_coord(lo.x, hi.x, iu, P.grid_nu);
  v = grid_coord(lo.y, hi.y, iv, P.grid_nv);
}

// Counters (optional, COUNT=true): 0 (query, segment) root tests, 1 hard pairs,
// 2 nodes, 3 evaluations, 4 leaves, 5 max depth, 6 warp-level skips (culled
// groups + pruned hierarchy subtrees), 7 on-boundary, 8 (query, SPAN) tests,
// 9 warp-record iterations of phase 1, 10 (query, SPAN) tests that descend
// (the rest substitute the run's chord), 11 (query, SEG) tests that substitute
// the chord (pruned, a5)
template <bool COUNT>
__device__ __forceinline__ void cnt_add(unsigned long long *c, int i, unsigned long long v) {
  if (COUNT && v) atomicAdd(c + i, v);
}

// Rational Bezier point by O(n) homogeneous Horner on c_j = C(n,j) w_j (P_j, 1)
// (Table 1):  sum_j c_j t^j (1-t)^(n-j)  =  (...(c_n t + c_{n-1} u) t
// + c_{n-2} u^2) t + ...,  u = 1-t.  t and u lie in [0,1] (no t/(1-t) blow-up,
// no branch on t), and the loop runs over the padded maximum degree with the
// zero coefficients above n, so every lane of a warp runs the same code
// whatever its segment's degree (the coefficient pairs load as 16-B vectors).
template <typename R>
__device__ __forceinline__ void eval_point(const BaseCold<R> *__restrict__ C, int n, R t, R &x, R &y) {
  const R u = R(1) - t;
  R cx[6], cy[6], cw[6];
  if constexpr (sizeof(R) == 8) {
#pragma unroll
    for (int j = 0; j < 6; j += 2) {
      const double2 a = __ldg(reinterpret_cast<const double2 *>(&C->cx[j]));
      const double2 b = __ldg(reinterpret_cast<const double2 *>(&C->cy[j]));
      const double2 c = __ldg(reinterpret_cast<const double2 *>(&C->cw[j]));
      cx[j] = a.x; cx[j + 1] = a.y; cy[j] = b.x; cy[j + 1] = b.y; cw[j] = c.x; cw[j + 1] = c.y;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 6; ++j) { cx[j] = __ldg(&C->cx[j]); cy[j] = __ldg(&C->cy[j]); cw[j] = __ldg(&C->cw[j]); }
  }
  R X = 0, Y = 0, W = 0, up = 1;
#pragma unroll
  for (int j = 5; j >= 0; --j) {
    X = X * t + cx[j] * up;
    Y = Y * t + cy[j] * up;
    W = W * t + cw[j] * up;
    up = (j <= n) ? up * u : up;
  }
  const R iw = R(1) / W;
  x = X * iw;
  y = Y * iw;
}

struct HardResult {
  int xsum;
  double fsum;   // radians (angle mode)
  bool ob;
};

// Span of the recursion node [ta, ta + 2^-d], d >= 1 (Eq. 2, with the
// tightest stored bound covering the node, R29): depth 1..3 nodes are unions
// of whole dyadic pieces -- tabulated min(2^-d max Bq, sum Lq) (R9); deeper
// nodes lie inside piece q: Bq[q] 2^-d.  One load, no per-node loop.
template <typename R>
__device__ __forceinline__ R node_span(const BaseCold<R> *__restrict__ C, int d, double ta) {
  if (d <= 3) {
    const int k = (int)(ta * (double)(1 << d));
    return (R)__ldg(&C->Sp[(1 << d) - 2 + k]);
  }
  return ldexp((R)__ldg(&C->Bq[(int)(ta * 8.0)]), -d);
}

// Alg. 1 line 3 without square roots: with r0 = d0^2, r1 = d1^2 and
// k = S^2 - r0 - r1,  d0 + d1 > S  <=>  k < 0 or 4 r0 r1 > k^2  (S > 0).  The
// rounding of either form is far inside the R5 margin folded into S.
#ifndef WN_HARD_SQRTFREE
#define WN_HARD_SQRTFREE 1
#endif
template <typename R>
__device__ __forceinline__ bool outside_ellipse(R r0, R r1, R S) {
#if WN_HARD_SQRTFREE
  const R k = S * S - r0 - r1;
  return k < R(0) || R(4) * r0 * r1 > k * k;
#else
  return dsqrt(r0) + dsqrt(r1) > S;
#endif
}

// Margin M of a face as R (fp32: rounded up, still a valid margin)
template <typename R>
__device__ __forceinline__ R margin_r(double M) {
  if constexpr (sizeof(R) == 8) return M;
  else return __double2float_ru(M);
}

// Split point of a copy: the base (stored) curve evaluated by Horner, then
// moved into the copy's frame (lift shift + copy translate, CopyFrame).
template <typename R>
__device__ __forceinline__ void eval_copy(const BaseCold<R> *__restrict__ C, int n, const CopyFrame &Fr, R t, R &x,
                                          R &y) {
  R x0, y0;
  eval_point(C, n, t, x0, y0);
  x = (R)Fr.X((double)x0);
  y = (R)Fr.Y((double)y0);
}

// One hard pair (query point q, emitted segment = copy record cr of base
// segment C) by Alg. 1 with an explicit stack of right end points (DESIGN.md
// 6).  The root is split immediately (phase 1 could not certify it as
// pruned).  All arithmetic in R, exact decisions; the copy's end points are
// lat(lat(x, k_s), k_g) exactly as the emission computed the hot chain points.
template <typename R, bool COUNT>
__device__ __noinline__ HardResult hard_pair(const BaseCold<R> *__restrict__ C, const CopyFrame Fr, R M, R qx, R qy,
                                             bool angle, R eps, int max_depth, unsigned long long *counters) {
  const int n = __ldg(&C->n);
  R stx[MAXD + 1], sty[MAXD + 1];
  int8_t std_[MAXD + 1];
  R Lx = (R)Fr.X(__ldg(&C->x0)) - qx, Ly = (R)Fr.Y(__ldg(&C->y0)) - qy;
  R rL = Lx * Lx + Ly * Ly;          // squared distances (no square roots, outside_ellipse)
  const R eps2 = eps * eps;
  stx[0] = (R)Fr.X(__ldg(&C->xn)) - qx;
  sty[0] = (R)Fr.Y(__ldg(&C->yn)) - qy;
  std_[0] = 0;
  int sp = 1;
  double ta = 0.0;   // node start: exact dyadic (double also for fp32 records)
  HardResult res{0, 0.0, false};
  bool root = true;
  unsigned long long nodes = 0, evals = 0, leaves = 0;
  int dmax = 0;
  while (sp > 0) {
    const R rx = stx[sp - 1], ry = sty[sp - 1];
    const int d = std_[sp - 1];
    const R rR = rx * rx + ry * ry;
    bool split;
    ++nodes;
    if (root) {
      split = true;
      root = false;
      if (rL < eps2 || rR < eps2) { res.ob = true; break; } // Alg. 1 line 1 on the root
    } else {
      if (rR < eps2) { res.ob = true; break; }              // Alg. 1 line 1
      const R span = node_span(C, d, ta) + M;                // Eq. 2 + margin (R5)
      split = !outside_ellipse(rL, rR, span);               // Alg. 1 line 3
    }
    if (!split) {                                           // chord substitution
      if (angle) res.fsum += (double)chord_angle(Lx, Ly, rx, ry);
      else res.xsum += xcount(Lx, Ly, rx, ry);
      ++leaves;
      Lx = rx; Ly = ry; rL = rR;
      ta += ldexp(1.0, -d);
      --sp;
    } else {
      if (d >= max_depth) { res.ob = true; break; }         // depth cap (R6)
      const double tm = ta + ldexp(1.0, -(d + 1));         // m = (a+b)/2
      R mx, my;
      eval_copy(C, n, Fr, (R)tm, mx, my);
      ++evals;
      std_[sp - 1] = (int8_t)(d + 1);
      stx[sp] = mx - qx;
      sty[sp] = my - qy;
      std_[sp] = (int8_t)(d + 1);
      ++sp;
      dmax = max(dmax, d + 1);
    }
  }
  if (COUNT) {
    cnt_add<COUNT>(counters, 2, nodes);
    cnt_add<COUNT>(counters, 3, evals);
    cnt_add<COUNT>(counters, 4, leaves);
    atomicMax(counters + 5, (unsigned long long)dmax);
  }
  return res;
}

__device__ __forceinline__ double nan_d() { return __longlong_as_double(0x7ff8000000000000LL); }

__device__ __forceinline__ uint8_t classify(double w, int rule) {
  const double r = w >= 0.0 ? floor(w + 0.5) : -floor(-w + 0.5);   // round half away (R10)
  return (rule == 0) ? (fabs(r) >= 1.0) : (r >= 1.0);
}

// fp32 distance |(dx,dy)|: r * rsqrt(r); 0 / overflow give NaN or inf, and every
// test below treats NaN as "not certified" (conservative).
__device__ __forceinline__ float fdist(float dx, float dy) {
  const float r = fmaf(dx, dx, dy * dy);
  return r * rsqrtf(r);
}

template <typename R>
__device__ __forceinline__ bool group_out(const Hot<R> &h, double px, double py);
template <>
__device__ __forceinline__ bool group_out<double>(const Hot<double> &h, double px, double py) {
  // fp32 box rounded outward vs the fp32-rounded point: RN is monotone, so a
  // point inside the exact box is never culled (exact-conservative)
  const float x = (float)px, y = (float)py, ymax = __int_as_float(__double2loint(h.x));
  return !(h.fx <= x && x <= h.fs && h.fy <= y && y <= ymax);
}
template <>
__device__ __forceinline__ bool group_out<float>(const Hot<float> &h, double px, double py) {
  const __half2 hi = *reinterpret_cast<const __half2 *>(&h.c);
  const float x = (float)px, y = (float)py;
  return !(h.a <= x && x <= __half2float(hi.x) && h.b <= y && y <= __half2float(hi.y));
}

// ---------------------------------------------------------------------------
// K3a: phase 1 of the query kernel.  One CTA (NTH threads) = one tile of up to
// QT = NTH queries of one face, one query per thread; the face's TMA-staged
// record program is swept in lock-step by all warps, so every record is one
// broadcast shared-memory read shared by the 32 queries of a warp.
// Records form, per chain, the path hierarchy of P:372-380 (pre-order SPAN
// nodes over SEG leaves): a warp skips a SPAN's subtree when every active lane
// is outside its ellipse.  Hard (query, segment) pairs go to the global queue.
// ---------------------------------------------------------------------------
template <typename R>
struct HotView;
template <>
struct HotView<double> {   // one 32-B record: two ld.shared.v4 at a 32-bit shared address
  float fx, fy, fs;
  uint32_t meta;
  double x, y;
  __device__ __forceinline__ void load(unsigned a) {
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(fx), "=f"(fy), "=f"(fs), "=r"(meta)
                 : "r"(a));
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(a + 16));
  }
};
template <>
struct HotView<float> {
  float fx, fy, fs;
  uint32_t meta;
  double x, y;   // fp32 records: (x, y) = (fx, fy) promoted
  __device__ __forceinline__ void load(unsigned a) {
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(fx), "=f"(fy), "=f"(fs), "=r"(meta)
                 : "r"(a));
    x = fx;
    y = fy;
  }
};

__device__ __forceinline__ bool group_out_v(const HotView<double> &h, float pxf, float pyf) {
  // as group_out<double>: fp32 comparisons, exact-conservative
  const float ymax = __int_as_float(__double2loint(h.x));
  return !(h.fx <= pxf && pxf <= h.fs && h.fy <= pyf && pyf <= ymax);
}
__device__ __forceinline__ bool group_out_v(const HotView<float> &h, float x, float y) {
  uint32_t c = __float_as_uint(h.fs);
  const __half2 hi = *reinterpret_cast<const __half2 *>(&c);
  return !(h.fx <= x && x <= __half2float(hi.x) && h.fy <= y && y <= __half2float(hi.y));
}

// omega(p, L) for a slanted line (K_SLINE): +1/2 iff p is left of the line
// through b along v = (p Tu, q Tv), i.e. cross(v, p - b) >= 0 (on L
// counts as left, R11).  Evaluated without contraction, in the order of the
// plain definition, so the decision is the correctly rounded one of that
// expression.
__device__ __forceinline__ bool sline_left(uint32_t meta, double bx, double by, double px, double py,
                                           const double *__restrict__ dom) {
  const int p = ((int)(meta << 12)) >> 20;
  const int q = ((int)meta) >> 20;
  const double vx = __dmul_rn((double)p, __ldg(dom + 1)), vy = __dmul_rn((double)q, __ldg(dom + 3));
  const double cr = __dsub_rn(__dmul_rn(vx, __dsub_rn(py, by)), __dmul_rn(vy, __dsub_rn(px, bx)));
  return cr >= 0.0;
}

// approximate fp32 |(dx,dy)| with flush-to-zero rsqrt (1 MUFU); a zero or
// overflowing argument gives NaN/inf and every filter test treats it as
// "not certified" (conservative)
__device__ __forceinline__ float fdist_ftz(float dx, float dy) {
  const float r = fmaf(dx, dx, dy * dy);
  float rs;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(rs) : "f"(r));
  return r * rs;
}

// intermediate flag values between phase 1 and k_finish / k_overflow
constexpr uint8_t FLAG_PENDING = 0xFF;    // hard pairs queued: k_finish classifies
constexpr uint8_t FLAG_OVERFLOW = 0xFE;   // a hard pair did not fit the queue: k_overflow recomputes

#ifndef WN_P1_INTEPI
#define WN_P1_INTEPI 1          // integer classification when the query met no line and no angle term
#endif
#ifndef WN_P1_QPIPE
#define WN_P1_QPIPE 1           // the next sub-tile's query points copied to shared memory (cp.async) during the sweep
#endif
constexpr int HWB = WN_P1_QPIPE ? 48 : 64;   // per-warp shared-memory buffer of hard pairs (flushed with one atomic)
constexpr int HCHUNK = 32;   // hard pairs a k_hard warp reserves per atomic (one per lane: small queues stay spread)
#ifndef WN_P1_PINF
#define WN_P1_PINF 1            // the query's fp32 coordinates pinned in registers
#endif
#ifndef WN_HARD_BPS
#define WN_HARD_BPS 8           // k_hard CTAs per SM (2 waves; 2 or 4 measured no better)
#endif
#ifndef WN_HARD_DYN
#define WN_HARD_DYN 0           // 1: dynamic fetching of hard pairs per warp (measured slower on C5); 0: static grid stride
#endif
constexpr int SP_BINS = 1024;   // Morton cells of the spatial regrouping (32 x 32)
constexpr int SP_COHERENT = 24; // mean warp-footprint perimeter (cells) above which a unit is regrouped

#ifndef WN_QPL
#define WN_QPL 1                // queries per thread in k_phase1 (1 or 2)
#endif
#ifndef WN_P1_ZIDX
#define WN_P1_ZIDX 1            // chain points as shared addresses of their records (not 2 doubles)
#endif

// exact point of the record at shared address a (fp64 records: (x, y) at +16;
// fp32 records: (fx, fy) at +0, promoted)
template <typename R>
__device__ __forceinline__ void zget(unsigned a, double &x, double &y) {
  if constexpr (sizeof(R) == 8) {
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(a + 16) : "memory");
  } else {
    float fx, fy;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(fx), "=f"(fy) : "r"(a) : "memory");
    x = fx;
    y = fy;
  }
}
// the address zget reads for a 16-B parking slot
template <typename R>
__device__ __forceinline__ unsigned zslot(unsigned slot) { return sizeof(R) == 8 ? slot - 16 : slot; }
// copy the point of record a into the parking slot; returns its zget address
template <typename R>
__device__ __forceinline__ unsigned zpark(unsigned a, unsigned slot) {
  if constexpr (sizeof(R) == 8) {
    double x, y;
    zget<R>(a, x, y);
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(slot), "d"(x), "d"(y) : "memory");
  } else {
    float fx, fy;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(fx), "=f"(fy) : "r"(a) : "memory");
    asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(slot), "f"(fx), "f"(fy) : "memory");
  }
  return zslot<R>(slot);
}
#ifndef WN_P1_MINB
#define WN_P1_MINB (WN_QPL == 1 ? 4 : 3)
#endif
constexpr int QPL = WN_QPL;
constexpr int QTK = QT * QPL;   // queries per sub-tile of k_phase1

// ANGLE: the build's angle_mode (every record of a handle carries the same F_ANGLE);
// GRID: implicit-grid batch (wn_query_grid) instead of explicit uv.
// Each thread evaluates QPL queries (QPL = 2: two independent query chains per
// record, the record load / decode / warp decisions shared by 64 queries).
template <typename R, bool COUNT, bool ANGLE, bool GRID>
__global__ void __launch_bounds__(NTH, WN_P1_MINB) k_phase1(QParams<R> P) {
  constexpr bool F64 = sizeof(R) == 8;
  // records per staged chunk: 32 KB, or 28 KB when the chain-point parking
  // slots (4.2 KB) must fit the 48-KB static shared memory too
  constexpr int RCH = (F64 ? 1024 : 2048) * (WN_P1_ZIDX ? (WN_P1_QPIPE ? 27 : 28) : 32) / 32;
  __shared__ __align__(128) Hot<R> s_rec[RCH];
  __shared__ HardEntry s_hb[NWARP][HWB];
  __shared__ __align__(8) uint64_t s_bar;
#if WN_P1_ZIDX
  __shared__ __align__(16) double2 s_park[NTH * QPL + NWARP];   // chain points parked across chunks
#endif
#if WN_P1_QPIPE
  __shared__ __align__(16) double2 s_q[NTH * QPL];               // the thread's query points of the next sub-tile
#endif

  if ((int)blockIdx.x >= *P.ntiles) return;               // uniform: no tile
  const Tile T = P.tiles[blockIdx.x];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int f = T.face;
  if (f < 0) {                                             // grid of an invalid face id: flag 3
    for (int i = t; i < T.qcnt; i += NTH) {
      P.winding[T.qbeg + i] = nan_d();
      P.flag[T.qbeg + i] = 3;
    }
    return;
  }
  const int rec0 = P.face_rec_off[f];
  const int nrec = P.face_rec_off[f + 1] - rec0;
  // a face program that fits one chunk is staged once and reused by every
  // sub-tile of the unit (the copy overlaps the first query loads)
  const bool single = nrec <= RCH;
  if (t == 0) {
    mbar_init(&s_bar, 1);
    fence_mbar_init();
    WN_DCHECK(nrec >= 0 && rec0 >= 0 && rec0 + nrec <= P.n_rec);
    if (single && nrec > 0) {
      fence_proxy_async_smem();
      mbar_arrive_expect_tx(&s_bar, (unsigned)(nrec * sizeof(Hot<R>)));
      tma_bulk_g2s(s_rec, P.hot + rec0, (unsigned)(nrec * sizeof(Hot<R>)), &s_bar);
    }
  }
  const uint8_t per = P.face_per[f];
  const double *dom = P.face_dom + 4 * f;
  const int unsorted = *P.unsorted;
  const int cold0 = P.face_cold_off[f];
  // spatial regrouping of explicit units (see below)
  __shared__ uint32_t s_hist[SP_BINS / 2];   // 16-bit counters, two per word
  __shared__ int s_wsum[NWARP];
  __shared__ int s_coh[2];                   // coherence probe: perimeter sum, warps
  __shared__ double s_v0;                    // row probe: v of the unit's first query
  __shared__ int s_nu;                       // row probe: first index with another v
  if (t < 2) s_coh[t] = 0;
  if (t == 0) s_nu = QTK;
  // implicit grid: a unit lies inside one grid (units are cut per grid), so the
  // grid index, its box and the cell steps are per-CTA values (kept in shared
  // memory, not in registers across the record loop)
  __shared__ double s_grid[4];   // u_lo, v_lo, (u_hi - u_lo) / nu, (v_hi - v_lo) / nv
  __shared__ int s_gloc0;
  if constexpr (GRID) {
    if (t == 0) {
      const int64_t g = T.qbeg / P.grid_n;
      s_gloc0 = (int)(T.qbeg - g * P.grid_n);
      const double2 lo = __ldg(P.grid_box + 2 * g), hi = __ldg(P.grid_box + 2 * g + 1);
      s_grid[0] = lo.x;
      s_grid[1] = lo.y;
      s_grid[2] = __ddiv_rn(__dsub_rn(hi.x, lo.x), (double)P.grid_nu);   // as in grid_coord
      s_grid[3] = __ddiv_rn(__dsub_rn(hi.y, lo.y), (double)P.grid_nv);
    }
  }
  const double eps = P.eps;
  // fp32-filter constant: a distance df > eps_c certifies d >= eps
  // (fp64 records; margins 2^-16 scale + 2^-17 relative)
  const float eps_c = F64 ? __double2float_ru((eps + P.face_M[f] * 0x1p24) * (1.0 + 0x1p-17)) : (float)eps;
  // shared address of the record buffer, opaque to the compiler so that it is
  // kept in a register instead of being recomputed in the inner loop
  unsigned sbase;
  asm volatile("mov.u32 %0, %1;" : "=r"(sbase) : "r"(smem_u32(s_rec)));
  unsigned phase = 0;
  int hn_ = 0;                   // entries in this warp's hard-pair buffer (warp-uniform)
  unsigned long long c_pairs = 0, c_hard = 0, c_cull = 0, c_span = 0, c_rec = 0, c_desc = 0, c_prn = 0;
  __syncthreads();               // barrier initialised
  // pend bits of the lane's current queries: 1 hard pairs queued, 2 one of them
  // overflowed the queue, 4 entries still in the warp buffer
  int pend[QPL];
#pragma unroll
  for (int k = 0; k < QPL; ++k) pend[k] = 0;

  // flush the warp's buffer to the global queue with one exact reservation.
  // Entries past the capacity mark their query FLAG_OVERFLOW (recomputed
  // exactly by k_overflow); the lane's own current queries also keep bit 2
  // because their final flags are written after this.
  auto flush = [&]() {
    __syncwarp();
    int b = 0;
    if (lane == 0) {
      // saturating reservation: once the queue is full the counter only
      // moves to cap + 1 (marks the overflow for k_overflow), so it can never
      // wrap however many pairs a batch attempts
      if (*reinterpret_cast<volatile int32_t *>(P.hq_count) >= P.hq_cap) {
        b = P.hq_cap;
        atomicMax(P.hq_count, P.hq_cap + 1);
      } else {
        b = atomicAdd(P.hq_count, hn_);
      }
    }
    b = __shfl_sync(0xffffffffu, b, 0);
    bool ovf = false;
    for (int i = lane; i < hn_; i += 32) {
      WN_DCHECK(i < HWB && s_hb[warp][i].q >= 0 && s_hb[warp][i].q < P.nq);
      if (b + i < P.hq_cap) {
        P.hq[b + i] = s_hb[warp][i];
      } else {
        P.flag[s_hb[warp][i].q] = FLAG_OVERFLOW;
        ovf = true;
      }
    }
    const bool any_ovf = __any_sync(0xffffffffu, ovf);
#pragma unroll
    for (int k = 0; k < QPL; ++k) {
      if (any_ovf && (pend[k] & 4)) pend[k] |= 2;
      pend[k] &= ~4;
    }
    __syncwarp();
    hn_ = 0;
  };

  // Spatial regrouping (explicit batches): the unit's queries are put in
  // Morton order of a 32 x 32 cell grid over the face's box (a counting sort
  // in shared memory, once per unit), so that each warp takes 32 QPL queries
  // that lie close together and agrees more often on pruning a span or
  // culling a group.  A permutation of whole queries: no value changes.  The
  // order goes to a per-unit scratch range (L2-resident), read per sub-tile.
  bool spatial = false;
  // queries of this thread within a sub-tile: query k of lane l of warp w is
  // at sub-tile position w 32 QPL + 32 k + l (given order, Morton order), or
  // (2-D tiles) in a bw x (32 QPL / bw) block of cells of the warp
  int lt[QPL];
#pragma unroll
  for (int k = 0; k < QPL; ++k) lt[k] = warp * 32 * QPL + 32 * k + lane;
  if constexpr (!GRID) {
    spatial = P.spatial && T.qcnt > 32;
    const float4 fb = spatial ? P.face_box[f] : make_float4(0.f, 0.f, 0.f, 0.f);
    {
      const float sx = fb.z > fb.x ? 32.f / (fb.z - fb.x) : 0.f, sy = fb.w > fb.y ? 32.f / (fb.w - fb.y) : 0.f;
      auto key_of = [&](int i, int32_t &qi_out) {
        const int32_t pos = (int32_t)T.qbeg + i;
        const int32_t qi = unsorted ? P.perm[pos] : pos;
        qi_out = qi;
        const double u = P.uv[2 * (int64_t)qi], v = P.uv[2 * (int64_t)qi + 1];
        if (!isfinite(u) || !isfinite(v)) return SP_BINS - 1;
        const double ur = (per & 1) ? reduce_coord(u, dom[0], dom[1]) : u;
        const double vr = (per & 2) ? reduce_coord(v, dom[2], dom[3]) : v;
        const int cx = min(max(__float2int_rd(((float)ur - fb.x) * sx), 0), 31);
        const int cy = min(max(__float2int_rd(((float)vr - fb.y) * sy), 0), 31);
        int mx = cx, my = cy;   // interleave 5 + 5 bits
        mx = (mx | (mx << 4)) & 0x0F0F; mx = (mx | (mx << 2)) & 0x3333; mx = (mx | (mx << 1)) & 0x5555;
        my = (my | (my << 4)) & 0x0F0F; my = (my | (my << 2)) & 0x3333; my = (my | (my << 1)) & 0x5555;
        return mx | (my << 1);
      };
      if (spatial) {
        // Coherence probe on the first QT queries in their given order: the
        // mean perimeter (in cells) of a warp's footprint.  Already coherent
        // input (e.g. row-major grids: a warp covers a short run of one row) is
        // left in its order -- regrouping it would cost more than it saves.
        {
          int cx = 0, cy = 0;
          bool ok = t < T.qcnt;
          if (ok) {
            int32_t q_;
            const int k = key_of(t, q_);
            // cell coordinates back from the Morton key
            int a = k & 0x5555, b = (k >> 1) & 0x5555;
            a = (a | (a >> 1)) & 0x3333; a = (a | (a >> 2)) & 0x0F0F; a = (a | (a >> 4)) & 0x00FF;
            b = (b | (b >> 1)) & 0x3333; b = (b | (b >> 2)) & 0x0F0F; b = (b | (b >> 4)) & 0x00FF;
            cx = a;
            cy = b;
          }
          const unsigned m = __ballot_sync(0xffffffffu, ok);
          if (m) {
            const unsigned x0 = __reduce_min_sync(0xffffffffu, ok ? (unsigned)cx : 255u);
            const unsigned x1 = __reduce_max_sync(0xffffffffu, ok ? (unsigned)cx : 0u);
            const unsigned y0 = __reduce_min_sync(0xffffffffu, ok ? (unsigned)cy : 255u);
            const unsigned y1 = __reduce_max_sync(0xffffffffu, ok ? (unsigned)cy : 0u);
            if (lane == 0) {
              atomicAdd(&s_coh[0], (int)((x1 - x0) + (y1 - y0)));
              atomicAdd(&s_coh[1], 1);
            }
          }
        }
        // Row probe: a unit that starts with whole rows of length nu (v constant
        // along a row; nu dividing QTK) -- a row-major tessellation grid -- is
        // mapped to 2-D warp tiles like wn_query_grid, without sorting
        double vt = 0.0;
        if (t < T.qcnt) {
          const int32_t pos = (int32_t)T.qbeg + t;
          vt = P.uv[2 * (int64_t)(unsorted ? P.perm[pos] : pos) + 1];
          if (t == 0) s_v0 = vt;
        }
        for (int i = t; i < SP_BINS / 2; i += NTH) s_hist[i] = 0;
        __syncthreads();
        if (t > 0 && t < T.qcnt && !(vt == s_v0)) atomicMin(&s_nu, t);
        __syncthreads();
        const int nu = s_nu;
        if (T.qcnt >= QTK && nu >= 8 && nu < QTK && QTK % nu == 0 && QTK / nu <= 32 * QPL) {
          const int bw = 32 * QPL / (QTK / nu);   // row-major unit: the same 2-D tiles as a grid
#pragma unroll
          for (int k = 0; k < QPL; ++k) {
            const int i = lane + 32 * k;
            lt[k] = (i / bw) * nu + warp * bw + i % bw;
          }
          spatial = false;
        } else {
          spatial = s_coh[0] > SP_COHERENT * s_coh[1];
        }
      }
    if (spatial) {
      // pass 1: key and rank within its cell -> scratch (key << 12 | rank)
#pragma unroll 4
      for (int i = t; i < T.qcnt; i += NTH) {
        int32_t q_;
        const int k = key_of(i, q_);
        const uint32_t old = atomicAdd(&s_hist[k >> 1], 1u << (16 * (k & 1)));
        P.skey[T.qbeg + i] = (k << 12) | (int)((old >> (16 * (k & 1))) & 0xFFFu);
      }
      __syncthreads();
      // exclusive scan of the SP_BINS counters: each thread owns SP_BINS / NTH
      constexpr int PER = SP_BINS / NTH;   // bins per thread (even)
      uint32_t c[PER];
      int tot = 0;
#pragma unroll
      for (int j = 0; j < PER; j += 2) {
        const uint32_t wv = s_hist[(t * PER + j) >> 1];
        c[j] = wv & 0xFFFFu;
        c[j + 1] = wv >> 16;
        tot += (int)(c[j] + c[j + 1]);
      }
      int incl = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int nb = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += nb;
      }
      if (lane == 31) s_wsum[warp] = incl;
      __syncthreads();
      int base = incl - tot;
#pragma unroll
      for (int w2 = 0; w2 < NWARP; ++w2) base += (w2 < warp) ? s_wsum[w2] : 0;
#pragma unroll
      for (int j = 0; j < PER; j += 2) {
        const uint32_t o0 = (uint32_t)base, o1 = (uint32_t)base + c[j];
        base += (int)(c[j] + c[j + 1]);
        s_hist[(t * PER + j) >> 1] = o0 | (o1 << 16);      // offsets <= 4096: no carry
      }
      __syncthreads();
      // pass 2: position = cell offset + rank in cell (no atomics, no reload of uv)
#pragma unroll 4
      for (int i = t; i < T.qcnt; i += NTH) {
        const int32_t pos = (int32_t)T.qbeg + i;
        const int kr = P.skey[pos];
        const int k = kr >> 12;
        const uint32_t off = (s_hist[k >> 1] >> (16 * (k & 1))) & 0xFFFFu;
        WN_DCHECK((int)off + (kr & 0xFFF) < T.qcnt);
        P.sorder[T.qbeg + (int)off + (kr & 0xFFF)] = unsorted ? P.perm[pos] : pos;
      }
      __syncthreads();   // the order (global, this CTA's range) is visible to the block
    }
    }
  }

  // Implicit grids whose rows tile a sub-tile (grid_blk > 0) give each warp a
  // compact bw x (32 QPL / bw) block of cells instead of a run of one row: the
  // warp's queries then lie close together, so they agree more often on
  // pruning a hierarchy span or culling a group (fewer warp-level descents).
  if constexpr (GRID) {
    const int bw = P.grid_blk;
    if (bw > 0) {
#pragma unroll
      for (int k = 0; k < QPL; ++k) {
        const int i = lane + 32 * k;
        lt[k] = (i / bw) * P.grid_nu + warp * bw + i % bw;
      }
    }
  }

#if WN_P1_QPIPE
  // Query pipeline (explicit batches whose position is the query index): while a
  // sub-tile is swept, each thread's point of the next one travels to its
  // shared-memory slot with an asynchronous 16-B copy, so the next prologue
  // does not wait for global memory.
  const bool qpipe = !GRID && !spatial && !unsorted && ((reinterpret_cast<uintptr_t>(P.uv) & 15) == 0);
#else
  constexpr bool qpipe = false;
#endif
  // one unit = up to QU queries of face f, processed QTK at a time
  for (int sub = 0; sub < T.qcnt; sub += QTK) {
    bool valid[QPL];
    int32_t qi[QPL];
    double px[QPL], py[QPL];
    float pxf[QPL], pyf[QPL];
#pragma unroll
    for (int k = 0; k < QPL; ++k) {
      valid[k] = sub + lt[k] < T.qcnt;
      const int32_t pos = (int32_t)(T.qbeg + sub) + lt[k];
      qi[k] = valid[k] ? (spatial ? P.sorder[pos] : unsorted ? P.perm[pos] : pos) : 0;
      WN_DCHECK(!valid[k] || (qi[k] >= 0 && qi[k] < P.nq));
      px[k] = 0.0;
      py[k] = 0.0;
      if (valid[k]) {
        double u, v;
        if constexpr (GRID) {
          const int loc = s_gloc0 + sub + lt[k];
          const int iv = loc / P.grid_nu, iu = loc - iv * P.grid_nu;
          u = __dadd_rn(s_grid[0], __dmul_rn((double)iu + 0.5, s_grid[2]));   // = grid_coord(), bit for bit
          v = __dadd_rn(s_grid[1], __dmul_rn((double)iv + 0.5, s_grid[3]));
        } else {
#if WN_P1_QPIPE
          if (qpipe && sub > 0) {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
            asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(u), "=d"(v) : "r"(smem_u32(&s_q[t * QPL + k])) : "memory");
          } else
#endif
          {
            u = P.uv[2 * (int64_t)qi[k]];
            v = P.uv[2 * (int64_t)qi[k] + 1];
          }
          // the next sub-tile's point: to this thread's shared slot (query
          // pipeline; issued after (u, v) left the slot), else to L2
          if (!spatial && !unsorted && sub + QTK + lt[k] < T.qcnt) {
#if WN_P1_QPIPE
            if (qpipe) {
              asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n\tcp.async.commit_group;" ::"r"(smem_u32(&s_q[t * QPL + k])),
                           "l"(P.uv + 2 * (int64_t)(pos + QTK)), "d"(u), "d"(v)
                           : "memory");
            } else
#endif
              asm volatile("prefetch.global.L2 [%0];" ::"l"(P.uv + 2 * (int64_t)(pos + QTK)));
          }
        }
        if (!isfinite(u) || !isfinite(v)) {
          P.winding[qi[k]] = nan_d();
          P.flag[qi[k]] = 3;
          valid[k] = false;
        } else {
          if (per & 1) u = reduce_coord(u, dom[0], dom[1]);
          if (per & 2) v = reduce_coord(v, dom[2], dom[3]);
          if (!F64) { u = (double)(float)u; v = (double)(float)v; }
          px[k] = u;
          py[k] = v;
        }
      }
      pxf[k] = (float)px[k];
      pyf[k] = (float)py[k];
#if WN_P1_PINF
      // opaque: kept in registers instead of re-derived from (px, py) with an
      // F2F.F32.F64 conversion in every record iteration
      asm volatile("" : "+f"(pxf[k]), "+f"(pyf[k]));
#endif
    }

    // per-query chain state: previous chain point (exact), its fp32 distance,
    // its side of the cut; and the group start A (warp-uniform, set by MOVE).
    // WN_P1_ZIDX: the points are kept as the shared address of the record
    // that holds them (read back only when a crossing is computed)
#if WN_P1_ZIDX
    unsigned zs[QPL], gs = sbase;
#define ZSET(k) (zs[k] = (unsigned)sp)
#define ZGET(k, X, Y) double X, Y; zget<R>(zs[k], X, Y)
#define GSET() (gs = (unsigned)sp)
#define GGET(X, Y) double X, Y; zget<R>(gs, X, Y)
#else
    double zx[QPL], zy[QPL];
    double gax = 0.0, gay = 0.0;
#define ZSET(k) (zx[k] = h.x, zy[k] = h.y)
#define ZGET(k, X, Y) const double X = zx[k], Y = zy[k]
#define GSET() (gax = h.x, gay = h.y)
#define GGET(X, Y) const double X = gax, Y = gay
#endif
    float cdf[QPL];
    int up[QPL];                   // side of the branch cut of the previous chain point (0/1)
    bool onb[QPL];
    int skip_end[QPL];             // query inactive (culled / pruned subtree) while gr < skip_end
    // xs: crossings in the low 16 bits, line half-turns (+-1 per LINE / SLINE
    // record) in the high 16 -- one register for both counts
    int xs[QPL];
    double fr[QPL];
#pragma unroll
    for (int k = 0; k < QPL; ++k) {
#if WN_P1_ZIDX
      zs[k] = sbase;
#else
      zx[k] = zy[k] = 0.0;
#endif
      cdf[k] = 0.f;
      up[k] = 0;
      onb[k] = false;
      skip_end[k] = 0;
      xs[k] = 0;
      fr[k] = 0.0;
      pend[k] = 0;
    }
    int gr = 0;                    // warp-uniform record cursor

    for (int cb = 0; cb < nrec; cb += RCH) {
      const int cn = min(RCH, nrec - cb);
      if (!single) {
        if (t == 0) {
          fence_proxy_async_smem();
          mbar_arrive_expect_tx(&s_bar, (unsigned)(cn * sizeof(Hot<R>)));
          tma_bulk_g2s(s_rec, P.hot + rec0 + cb, (unsigned)(cn * sizeof(Hot<R>)), &s_bar);
        }
        while (!mbar_try_wait(&s_bar, phase)) {
        }
        phase ^= 1u;
      } else if (sub == 0) {
        while (!mbar_try_wait(&s_bar, 0)) {
        }
      }
      const int ce = cb + cn;
      // the record cursor and the queries' subtree ends as shared addresses
      // within this chunk (converted back to record indices at its end)
      constexpr int RB = (int)sizeof(Hot<R>);
      int sp = (int)sbase + (gr - cb) * RB;                    // shared address of record gr
      int sse[QPL];                                            // query inactive while sp < sse
#pragma unroll
      for (int k = 0; k < QPL; ++k) sse[k] = (int)sbase + (skip_end[k] - cb) * RB;
      const int spe = (int)sbase + cn * RB;
      while (sp < spe) {
        HotView<R> h;
        WN_DCHECK(sp >= (int)sbase && ((sp - (int)sbase) % RB) == 0);
        h.load((unsigned)sp);
        const uint32_t meta = h.meta;
        const uint32_t kind = meta & 0xFu;
        WN_DCHECK(kind <= K_SLINE && kind != 2u);
        bool act[QPL];
#pragma unroll
        for (int k = 0; k < QPL; ++k) act[k] = valid[k] && sp >= sse[k];
        if (COUNT && lane == 0) ++c_rec;
        if (__builtin_expect((meta & 0xEu) == 0u, 1)) {   // SEG (0) or SPAN (1)
          // a4: root eps-test and ellipse test (Alg. 1 lines 1-3, Eq. 1, R9,
          // R5) for SEG; the path-hierarchy bound Omega_{j,k} (span =
          // sum of root spans) for SPAN.  The fp32 filter certifies "outside the
          // ellipse, d >= eps"; a crossing / hard / uncertain query takes the
          // exact slow path.
          int u1[QPL];
          float df[QPL];
          bool pr[QPL];
#pragma unroll
          for (int k = 0; k < QPL; ++k) {
            if constexpr (F64) {
              u1[k] = h.y >= py[k] ? 1 : 0;                        // exact side of the branch cut
              df[k] = fdist_ftz(h.fx - pxf[k], h.fy - pyf[k]);
            } else {
              u1[k] = h.fy >= pyf[k] ? 1 : 0;
              const float dx = h.fx - pxf[k], dy = h.fy - pyf[k];
              df[k] = sqrtf(dx * dx + dy * dy);
            }
            pr[k] = cdf[k] + df[k] > h.fs && df[k] > eps_c;        // certified outside, end point >= eps
          }
          if (meta & 1u) {                                       // K_SPAN
            // descend unless every active query prunes the whole run
            bool descend = false;
#pragma unroll
            for (int k = 0; k < QPL; ++k) {
              if (COUNT && act[k]) ++c_span;
              if (COUNT && act[k] && !pr[k]) ++c_desc;
              descend |= act[k] && !pr[k];
            }
            if (!__any_sync(0xffffffffu, descend)) {
              // every active query substitutes the run's chord (homotopy)
#pragma unroll
              for (int k = 0; k < QPL; ++k) {
                if (act[k] && (u1[k] != up[k] || ANGLE)) {     // (a plain branch: uniform when no query crosses)
                  ZGET(k, zxk, zyk);
                  if (ANGLE) fr[k] += (double)chord_angle(zxk - px[k], zyk - py[k], h.x - px[k], h.y - py[k]);
                  else xs[k] += xcount(zxk - px[k], zyk - py[k], h.x - px[k], h.y - py[k]);
                }
                if (act[k]) { ZSET(k); cdf[k] = df[k]; up[k] = u1[k]; }
              }
              sp += (int)(meta >> 8) * RB;
              if (COUNT && lane == 0) ++c_cull;
            } else {
#pragma unroll
              for (int k = 0; k < QPL; ++k) {
                if (act[k] && pr[k]) {
                  // this query prunes the run: chord now, inactive for the subtree
                  if (ANGLE || u1[k] != up[k]) {
                    ZGET(k, zxk, zyk);
                    if (ANGLE) fr[k] += (double)chord_angle(zxk - px[k], zyk - py[k], h.x - px[k], h.y - py[k]);
                    else xs[k] += xcount(zxk - px[k], zyk - py[k], h.x - px[k], h.y - py[k]);
                  }
                  ZSET(k); cdf[k] = df[k]; up[k] = u1[k];
                  sse[k] = sp + RB + (int)(meta >> 8) * RB;
                }
              }
            }
          } else {
            bool hard[QPL];
#pragma unroll
            for (int k = 0; k < QPL; ++k) {
              hard[k] = false;
              if (act[k] && (!pr[k] || u1[k] != up[k] || ANGLE)) {   // (a plain branch; the ballot below is the one vote)
                if (!(df[k] > eps_c)) {                              // filter cannot certify d >= eps
                  if constexpr (F64) {
                    const double dx = h.x - px[k], dy = h.y - py[k];
                    onb[k] |= sqrt(dx * dx + dy * dy) < eps;
                  } else {
                    onb[k] |= df[k] < (float)eps;
                  }
                }
                if (cdf[k] + df[k] > h.fs && !onb[k]) {              // pruned: chord (a5)
                  if (ANGLE || u1[k] != up[k]) {
                    ZGET(k, zxk, zyk);
                    if (ANGLE) fr[k] += (double)chord_angle(zxk - px[k], zyk - py[k], h.x - px[k], h.y - py[k]);
                    else xs[k] += xcount(zxk - px[k], zyk - py[k], h.x - px[k], h.y - py[k]);
                  }
                } else {
                  hard[k] = !onb[k];                                 // exact recursion in phase 2
                }
              }
            }
            unsigned m[QPL];
            int cnt = 0;
#pragma unroll
            for (int k = 0; k < QPL; ++k) {
              m[k] = __ballot_sync(0xffffffffu, hard[k]);
              cnt += __popc(m[k]);
            }
            if (cnt) {
              if (hn_ + cnt > HWB) flush();
              int basek = hn_;
#pragma unroll
              for (int k = 0; k < QPL; ++k) {
                if (hard[k]) {
                  HardEntry H;
                  H.px = px[k];
                  H.py = py[k];
                  H.q = qi[k];
                  H.c = (uint32_t)(cold0 + (int)(meta >> 8)) | (ANGLE ? 0x80000000u : 0u);
                  WN_DCHECK(hn_ + cnt <= HWB && (int)(meta >> 8) >= 0 && cold0 + (int)(meta >> 8) < P.n_copy);
                  s_hb[warp][basek + __popc(m[k] & ((1u << lane) - 1u))] = H;
                  pend[k] |= 1 | 4;
                  if (COUNT) ++c_hard;
                }
                basek += __popc(m[k]);
              }
              hn_ += cnt;
            }
#pragma unroll
            for (int k = 0; k < QPL; ++k) {
              if (act[k]) { ZSET(k); cdf[k] = df[k]; up[k] = u1[k]; }
              if (COUNT && act[k]) ++c_pairs;
              if (COUNT && act[k] && !hard[k] && !onb[k]) ++c_prn;     // chord substituted (a5)
            }
          }
        } else if (kind == K_MOVE || kind == K_MOVEG) {
#pragma unroll
          for (int k = 0; k < QPL; ++k) {
            const double nx = h.x - px[k], ny = h.y - py[k];
            float nd;
            if constexpr (F64) nd = fdist_ftz(h.fx - pxf[k], h.fy - pyf[k]);
            else nd = sqrtf((float)(nx * nx + ny * ny));
            if (act[k]) {
              if (!(nd > eps_c)) onb[k] |= F64 ? (sqrt(nx * nx + ny * ny) < eps) : (nd < (float)eps);
              if (kind == K_MOVEG && !ANGLE) {
                // gap chord Z -> A': -omega(p,Z,A') + its crossing
                ZGET(k, zxk, zyk);
                const double ax = zxk - px[k], ay = zyk - py[k];
                const double cr = canon_cross(ax, ay, nx, ny);
                fr[k] -= atan2(cr, ax * nx + ay * ny);
                xs[k] += xcount_exact(ax, ay, nx, ny, cr);
              }
            }
            ZSET(k); cdf[k] = nd;
            up[k] = (F64 ? (h.y >= py[k]) : (h.fy >= pyf[k])) ? 1 : 0;
          }
          if (kind == K_MOVE) GSET();
        } else if (kind == K_GROUP) {
          // copy-group / closed-loop cull: p outside the group's box => exactly 0
          bool out[QPL], all_out = true;
#pragma unroll
          for (int k = 0; k < QPL; ++k) {
            out[k] = !act[k] || group_out_v(h, pxf[k], pyf[k]);
            all_out &= out[k];
          }
          const int skip = (int)(meta >> 8);
          if (__all_sync(0xffffffffu, all_out)) {
            sp += skip * RB;
            if (COUNT && lane == 0) ++c_cull;
          } else {
#pragma unroll
            for (int k = 0; k < QPL; ++k)
              if (out[k] && act[k]) sse[k] = sp + RB + skip * RB;
          }
        } else if (kind == K_LINE) {
          // omega(p,L) = +-1/2, p on L counts as left (R11)
#pragma unroll
          for (int k = 0; k < QPL; ++k) {
            const double q = (meta & F_AXISV) ? px[k] : py[k];
            const bool left = (meta & F_GE) ? (q >= h.x) : (q <= h.x);
            if (act[k]) xs[k] += left ? (1 << 16) : -(1 << 16);
          }
        } else if (kind == K_SLINE) {
#pragma unroll
          for (int k = 0; k < QPL; ++k)
            if (act[k]) xs[k] += sline_left(meta, h.x, h.y, px[k], py[k], dom) ? (1 << 16) : -(1 << 16);
        } else if (kind == K_XCH || kind == K_NCH || kind == K_CLOSEG) {
#pragma unroll
          for (int k = 0; k < QPL; ++k) {
            if (act[k]) {
              ZGET(k, zxk, zyk);
              GGET(gxk, gyk);
              const double cx = zxk - px[k], cy = zyk - py[k], ax = gxk - px[k], ay = gyk - py[k];
              if (kind == K_XCH) {
                xs[k] -= xcount_exact(ax, ay, cx, cy, canon_cross(ax, ay, cx, cy));
              } else if (kind == K_NCH) {
                fr[k] -= chord_angle(ax, ay, cx, cy);
              } else {
                const double cr = canon_cross(cx, cy, ax, ay);
                fr[k] -= atan2(cr, cx * ax + cy * ay);
                xs[k] += xcount_exact(cx, cy, ax, ay, cr);
              }
            }
          }
        }
        sp += RB;
      }
      gr = cb + (sp - (int)sbase) / RB;
#pragma unroll
      for (int k = 0; k < QPL; ++k) skip_end[k] = cb + (sse[k] - (int)sbase) / RB;
#if WN_P1_ZIDX
      if (!single) {
        // the chunk is about to be overwritten: chain points that still live in
        // it move to this thread's (warp's) parking slot
        const unsigned lo = sbase, hi = sbase + (unsigned)(RCH * RB);
#pragma unroll
        for (int k = 0; k < QPL; ++k)
          if (zs[k] >= lo && zs[k] < hi) zs[k] = zpark<R>(zs[k], smem_u32(&s_park[t * QPL + k]));
        if (gs >= lo && gs < hi) {
          const unsigned slot = smem_u32(&s_park[NTH * QPL + warp]);
          __syncwarp();
          if (lane == 0) zpark<R>(gs, slot);
          __syncwarp();
          gs = zslot<R>(slot);
        }
      }
#endif
      // all warps done with this chunk before it is overwritten (multi-chunk faces)
      if (!single && (ce < nrec || sub + QTK < T.qcnt)) __syncthreads();
    }

#undef ZSET
#undef ZGET
#undef GSET
#undef GGET
    // ---- a8 (phase-1 part): reduce, classify or hand over to phase 2 ----
#pragma unroll
    for (int k = 0; k < QPL; ++k) {
      if (valid[k]) {
        if (onb[k]) {
          P.winding[qi[k]] = nan_d();
          P.flag[qi[k]] = 2;
          if (COUNT) atomicAdd(P.counters + 7, 1ull);
        } else {
          double w;
          uint8_t fl;
          const int xc = (int)(int16_t)(xs[k] & 0xFFFF), halves = (xs[k] - xc) >> 16;
          if (WN_P1_INTEPI && halves == 0 && fr[k] == 0.0) {
            // closed loops only: omega is the integer crossing count (the same
            // bits as the general formula, without its double-precision rounding)
            w = (double)xc;
            fl = (P.rule == 0) ? (xc != 0) : (xc >= 1);
          } else {
            w = (double)xc + 0.5 * (double)halves + fr[k] * (1.0 / TWO_PI);
            fl = classify(w, P.rule);
          }
          P.winding[qi[k]] = w;
          P.flag[qi[k]] = (pend[k] & 2) ? FLAG_OVERFLOW : (pend[k] & 1) ? FLAG_PENDING : fl;
        }
      }
    }
  }
  if (hn_) flush();   // entries of finished queries: overflow marks their flags directly
  if (COUNT) {
    cnt_add<COUNT>(P.counters, 0, c_pairs);
    cnt_add<COUNT>(P.counters, 1, c_hard);
    cnt_add<COUNT>(P.counters, 6, c_cull);
    cnt_add<COUNT>(P.counters, 8, c_span);
    cnt_add<COUNT>(P.counters, 9, c_rec);
    cnt_add<COUNT>(P.counters, 10, c_desc);
    cnt_add<COUNT>(P.counters, 11, c_prn);
  }
}

// ---------------------------------------------------------------------------
// K3b: phase 2 -- every queued hard pair, grid-strided; results are added to
// the partial winding numbers (crossing mode: integers, exact in any order).
// ---------------------------------------------------------------------------
template <typename R, bool COUNT>
__global__ void __launch_bounds__(256) k_hard(QParams<R> P) {
  // Each lane runs Alg. 1 on one pair at a time as a state machine that
  // advances ONE recursion node per loop iteration; as soon as its pair ends it
  // takes the next one from the queue (dynamic fetching: one atomic per warp
  // for all its free lanes), so lanes stay busy until the queue is drained and
  // a warp waits for its slowest lane only at the very end (the recursion
  // depth is data dependent).  Same decisions and arithmetic as hard_pair().
  const int total = min(*P.hq_count, P.hq_cap);
  const R eps = (R)P.eps;
  const int max_depth = P.max_depth;
  const int lane = threadIdx.x & 31;
  bool drained = false;          // warp-uniform: the queue returned no more pairs
  int wb = 0, we = 0;            // warp-uniform: pairs [wb, we) reserved by this warp, not yet handed out
  int i = WN_HARD_DYN ? total : (int)(blockIdx.x * blockDim.x + threadIdx.x);   // this lane's next pair (total: none)
  R stx[MAXD + 1], sty[MAXD + 1];
  int8_t std_[MAXD + 1];
  const BaseCold<R> *C = nullptr;
  CopyFrame Fr{0.0, 0.0, 0.0, 0.0};
  R qx = 0, qy = 0, M = 0, Lx = 0, Ly = 0, rL = 0;     // rL: squared distance to the left end
  const R eps2 = eps * eps;
  int n = 0, sp = 0, xsum = 0, q = 0;
  double ta = 0.0, fsum = 0.0;
  bool live = false, root = false, angle = false;
  unsigned long long nodes = 0, evals = 0, leaves = 0;
  int dmax = 0;
  while (true) {
    if (WN_HARD_DYN && !drained) {
      // hand the warp's reserved pairs to its free lanes; reserve HCHUNK more
      // (one atomic per warp per HCHUNK pairs) when they run out
      unsigned freem = __ballot_sync(0xffffffffu, !live && i >= total);
      while (freem) {
        if (wb >= we) {
          int base = 0;
          if (lane == 0) base = atomicAdd(P.hq_next, HCHUNK);
          base = __shfl_sync(0xffffffffu, base, 0);
          wb = base;
          we = min(base + HCHUNK, total);
          if (wb >= we) { drained = true; break; }
        }
        const int avail = we - wb;
        const int rank = __popc(freem & ((1u << lane) - 1u));
        if (((freem >> lane) & 1u) && rank < avail) i = wb + rank;
        wb += min(__popc(freem), avail);
        freem = __ballot_sync(0xffffffffu, !live && i >= total);
      }
    }
    if (!__any_sync(0xffffffffu, live || i < total)) break;
    if (!live) {
      if (i >= total) continue;
      const HardEntry H = P.hq[i];
      angle = H.c >> 31;
      WN_DCHECK((int)(H.c & 0x7fffffffu) < P.n_copy && H.q >= 0 && H.q < P.nq);
      const CopyRec cr = P.copy[H.c & 0x7fffffffu];
      WN_DCHECK(cr.s >= 0 && cr.s < P.n_base);
      C = P.cold + cr.s;
      Fr = copy_frame(cr, P.face_dom);
      qx = (R)H.px;
      qy = (R)H.py;
      q = H.q;
      M = margin_r<R>(__ldg(P.face_M + cr.face));
      n = __ldg(&C->n);
      Lx = (R)Fr.X(__ldg(&C->x0)) - qx;
      Ly = (R)Fr.Y(__ldg(&C->y0)) - qy;
      rL = Lx * Lx + Ly * Ly;
      stx[0] = (R)Fr.X(__ldg(&C->xn)) - qx;
      sty[0] = (R)Fr.Y(__ldg(&C->yn)) - qy;
      std_[0] = 0;
      sp = 1;
      ta = 0.0;
      xsum = 0;
      fsum = 0.0;
      root = true;
      live = true;
    }
    // one node [ta, ta + 2^-d] with right end point (rx, ry), top of the stack
    const R rx = stx[sp - 1], ry = sty[sp - 1];
    const int d = std_[sp - 1];
    const R rR = rx * rx + ry * ry;
    bool split, ob;
    ++nodes;
    if (root) {
      root = false;
      ob = rL < eps2 || rR < eps2;                          // Alg. 1 line 1 on the root
      split = true;
    } else {
      ob = rR < eps2;                                       // Alg. 1 line 1
      const R span = node_span(C, d, ta) + M;                // Eq. 2 + margin (R5)
      split = !outside_ellipse(rL, rR, span);               // Alg. 1 line 3
    }
    bool done = ob;
    if (!ob && split && d >= max_depth) { ob = true; done = true; }   // depth cap (R6)
    if (!done) {
      if (!split) {                                         // chord substitution
        if (angle) fsum += (double)chord_angle(Lx, Ly, rx, ry);
        else xsum += xcount(Lx, Ly, rx, ry);
        ++leaves;
        Lx = rx; Ly = ry; rL = rR;
        ta += ldexp(1.0, -d);
        done = --sp == 0;
      } else {
        const double tm = ta + ldexp(1.0, -(d + 1));       // m = (a+b)/2
        R mx, my;
        eval_copy(C, n, Fr, (R)tm, mx, my);
        ++evals;
        WN_DCHECK(sp <= MAXD);
        std_[sp - 1] = (int8_t)(d + 1);
        stx[sp] = mx - qx;
        sty[sp] = my - qy;
        std_[sp] = (int8_t)(d + 1);
        ++sp;
        dmax = max(dmax, d + 1);
      }
    }
    if (done) {
      double *w = P.winding + q;
      if (ob) {
        atomicExch(reinterpret_cast<unsigned long long *>(w), 0x7ff8000000000000ULL);
      } else {
        const double add = (double)xsum + fsum * (1.0 / TWO_PI);
        if (add != 0.0) atomicAdd(w, add);
      }
      live = false;
      i = WN_HARD_DYN ? total : i + (int)(gridDim.x * blockDim.x);   // fetch again / static grid stride
    }
  }
  if (COUNT) {
    cnt_add<COUNT>(P.counters, 2, nodes);
    cnt_add<COUNT>(P.counters, 3, evals);
    cnt_add<COUNT>(P.counters, 4, leaves);
    atomicMax(P.counters + 5, (unsigned long long)dmax);
  }
}

// K3d: queries whose hard pairs overflowed the global queue: the whole record
// program again for that query, exact root tests against the (valid, inflated)
// stored span and the recursion inline.  Normally never has work.
template <typename R>
__global__ void k_overflow(QParams<R> P, const int32_t *__restrict__ face_id, int64_t n) {
  if (*P.hq_count <= P.hq_cap) return;   // nothing overflowed (uniform)
  for (int64_t qi = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; qi < n; qi += (int64_t)gridDim.x * blockDim.x) {
    if (P.flag[qi] != FLAG_OVERFLOW) continue;
    double u, v;
    int f;
    if (P.grid_box) { grid_point(P, qi, u, v); f = P.grid_face[qi / P.grid_n]; }
    else { f = face_id[qi]; u = P.uv[2 * (int64_t)qi]; v = P.uv[2 * (int64_t)qi + 1]; }
    const uint8_t per = P.face_per[f];
    const double *dom = P.face_dom + 4 * f;
    if (per & 1) u = reduce_coord(u, dom[0], dom[1]);
    if (per & 2) v = reduce_coord(v, dom[2], dom[3]);
    if (sizeof(R) == 4) { u = (double)(float)u; v = (double)(float)v; }
    const int rec0 = P.face_rec_off[f], rec1 = P.face_rec_off[f + 1];
    const CopyRec *copy_face = P.copy + P.face_cold_off[f];
    double cx = 0, cy = 0, cd = 0, ax = 0, ay = 0, fr = 0;
    int xs = 0, halves = 0;
    bool ob = false;
    for (int r = rec0; r < rec1 && !ob; ++r) {
      const Hot<R> h = P.hot[r];
      const uint32_t meta = h.meta, kind = meta & 0xFu;
      double hx, hy, hs;
      if constexpr (sizeof(R) == 8) { hx = h.x; hy = h.y; hs = h.fs; } else { hx = h.a; hy = h.b; hs = h.c; }
      if (kind == K_SPAN) continue;   // hierarchy node: always descend (exact, leaves only)
      if (kind == K_SEG || kind == K_MOVE || kind == K_MOVEG) {
        const double nx = hx - u, ny = hy - v, nd = sqrt(nx * nx + ny * ny);
        if (nd < P.eps) { ob = true; break; }
        if (kind == K_SEG) {
          if (cd + nd > hs) {
            if (meta & F_ANGLE) fr += chord_angle(cx, cy, nx, ny);
            else xs += xcount(cx, cy, nx, ny);
          } else {
            const CopyRec cr = copy_face[meta >> 8];
            const HardResult res = hard_pair<R, false>(P.cold + cr.s, copy_frame(cr, P.face_dom),
                                                       margin_r<R>(P.face_M[cr.face]), (R)u, (R)v,
                                                       (meta & F_ANGLE) != 0, (R)P.eps, P.max_depth, nullptr);
            if (res.ob) { ob = true; break; }
            xs += res.xsum;
            fr += res.fsum;
          }
        } else if (kind == K_MOVEG && !(meta & F_ANGLE)) {
          const double cr = canon_cross(cx, cy, nx, ny);
          fr -= atan2(cr, cx * nx + cy * ny);
          xs += xcount_exact(cx, cy, nx, ny, cr);
        }
        if (kind == K_MOVE) { ax = nx; ay = ny; }
        cx = nx; cy = ny; cd = nd;
      } else if (kind == K_GROUP) {
        if (group_out<R>(h, u, v)) r += (int)(meta >> 8);
      } else if (kind == K_LINE) {
        const double q = (meta & F_AXISV) ? u : v;
        halves += ((meta & F_GE) ? (q >= hx) : (q <= hx)) ? 1 : -1;
      } else if (kind == K_SLINE) {
        halves += sline_left(meta, hx, hy, u, v, dom) ? 1 : -1;
      } else if (kind == K_XCH) {
        xs -= xcount_exact(ax, ay, cx, cy, canon_cross(ax, ay, cx, cy));
      } else if (kind == K_NCH) {
        fr -= chord_angle(ax, ay, cx, cy);
      } else if (kind == K_CLOSEG) {
        const double cr = canon_cross(cx, cy, ax, ay);
        fr -= atan2(cr, cx * ax + cy * ay);
        xs += xcount_exact(cx, cy, ax, ay, cr);
      }
    }
    if (ob) {
      P.winding[qi] = nan_d();
      P.flag[qi] = 2;
    } else {
      const double w = (double)xs + 0.5 * (double)halves + fr * (1.0 / TWO_PI);
      P.winding[qi] = w;
      P.flag[qi] = classify(w, P.rule);
    }
  }
}

// K3c: classify the queries that had hard pairs (a8): every FLAG_PENDING entry
// of the flag array (4 flags per thread when the array is word aligned)
__device__ __forceinline__ uint8_t finish_one(uint8_t fl, const double *__restrict__ winding, int64_t q, int rule,
                                              unsigned long long *counters) {
  if (fl != FLAG_PENDING) return fl;
  const double w = winding[q];
  if (isnan(w)) {
    if (counters) atomicAdd(counters + 7, 1ull);
    return 2;
  }
  return classify(w, rule);
}

__global__ void k_finish(int64_t n, const double *__restrict__ winding, uint8_t *__restrict__ flag, int rule,
                         unsigned long long *counters) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (((uintptr_t)flag & 15) == 0) {
    const int64_t nv = n >> 4;
    uint4 *fv = reinterpret_cast<uint4 *>(flag);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += stride) {
      uint4 v = fv[i];
      if (((v.x | v.y | v.z | v.w) & 0x80808080u) == 0) continue;   // final flags are 0..3
      // all 16 windings in flight at once (a pending group has several)
      // the windings of the pending entries only (predicated loads, all in flight)
      uint32_t w[4] = {v.x, v.y, v.z, v.w};
      double wv[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const bool pk = ((w[k >> 2] >> (8 * (k & 3))) & 0xFFu) == FLAG_PENDING;
        wv[k] = pk ? winding[16 * i + k] : 0.0;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint32_t o = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          uint8_t fl = (uint8_t)(w[j] >> (8 * k));
          if (fl == FLAG_PENDING) {
            const double x = wv[4 * j + k];
            if (isnan(x)) {
              fl = 2;
              if (counters) atomicAdd(counters + 7, 1ull);
            } else {
              fl = classify(x, rule);
            }
          }
          o |= (uint32_t)fl << (8 * k);
        }
        w[j] = o;
      }
      fv[i] = make_uint4(w[0], w[1], w[2], w[3]);
    }
    for (int64_t q = (nv << 4) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += stride)
      flag[q] = finish_one(flag[q], winding, q, rule, counters);
  } else {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += stride)
      flag[q] = finish_one(flag[q], winding, q, rule, counters);
  }
}

// K3c over the hard-pair queue instead of the flag array: a query is PENDING
// only if all its hard pairs are in the queue, so visiting the queue's entries
// reaches every PENDING flag (1.8M entries instead of 82M flags on C5).  Several
// entries of one query write the same final flag (idempotent).
__global__ void k_finish_q(const HardEntry *__restrict__ hq, const int32_t *__restrict__ hq_count, int32_t hq_cap,
                           const double *__restrict__ winding, uint8_t *__restrict__ flag, int rule) {
  const int total = min(*hq_count, hq_cap);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int32_t q = hq[i].q;
    if (flag[q] == FLAG_PENDING) {
      const double w = winding[q];
      flag[q] = isnan(w) ? (uint8_t)2 : classify(w, rule);
    }
  }
}

// ---------------------------------------------------------------------------
// K4: bucketing by face (a3).  Histogram with warp-aggregated atomics and a
// sortedness flag; scatter only when the batch is not grouped by face.
// ---------------------------------------------------------------------------
// Histogram by runs: the count of face f is the sum over maximal runs of f of
// (end - start), so each run adds -start at its first and end at its last
// element -- two atomics per run (a face-sorted batch: two per face).  Four ids
// per thread (16-B loads when aligned); run neighbours across threads via
// shuffles, across warps from global memory.  Invalid ids are flagged (3) and
// belong to no run.
__device__ __forceinline__ int hist_key(int f, int n_faces) { return (f >= 0 && f < n_faces) ? f : -1; }

__global__ void k_hist(int64_t n, const int32_t *__restrict__ face_id, int32_t n_faces,
                       int32_t *__restrict__ cnt, int32_t *__restrict__ unsorted,
                       double *__restrict__ winding, uint8_t *__restrict__ flag) {
  constexpr int G = 16;  // ids per thread (four 16-B loads in flight)
  const bool vec = ((uintptr_t)face_id & 15) == 0;
  const int64_t ng = (n + G - 1) / G;
  const int lane = threadIdx.x & 31;
  bool uns = false;
  for (int64_t g0 = blockIdx.x * (int64_t)blockDim.x; g0 < ng; g0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = g0 + threadIdx.x;
    const int64_t i0 = g * G;
    int id[G];
    if (g < ng && vec && i0 + G - 1 < n) {
#pragma unroll
      for (int k = 0; k < G; k += 4) {
        const int4 v = *reinterpret_cast<const int4 *>(face_id + i0 + k);
        id[k] = v.x; id[k + 1] = v.y; id[k + 2] = v.z; id[k + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int k = 0; k < G; ++k) id[k] = (g < ng && i0 + k < n) ? face_id[i0 + k] : INT32_MIN;
    }
    // raw neighbours: previous id (i0-1) and next id (i0+G)
    int prv = __shfl_up_sync(0xffffffffu, id[G - 1], 1);
    int nxt = __shfl_down_sync(0xffffffffu, id[0], 1);
    if (lane == 0) prv = (g < ng && i0 > 0) ? face_id[i0 - 1] : INT32_MIN;
    if (lane == 31 || g + 1 >= ng) nxt = (g < ng && i0 + G < n) ? face_id[i0 + G] : INT32_MIN;
    // fast path: a whole group inside one run of a valid face id (the common
    // case, runs are a face's queries) -- no boundary, no atomic, sorted
    int dif = (prv ^ id[0]) | (nxt ^ id[0]);
#pragma unroll
    for (int k = 1; k < G; ++k) dif |= id[k] ^ id[0];
    if (dif == 0 && g < ng && i0 > 0 && i0 + G < n && hist_key(id[0], n_faces) >= 0) continue;
    if (g < ng) {
#pragma unroll
      for (int k = 0; k < G; ++k) {
        const int64_t i = i0 + k;
        if (i >= n) break;
        const int f = id[k];
        const int pf = k ? id[k - 1] : prv;
        const int nf_ = (k < G - 1 && i + 1 < n) ? id[k + 1] : nxt;
        if (i > 0 && pf > f) uns = true;
        const int key = hist_key(f, n_faces);
        if (key < 0) {
          winding[i] = __longlong_as_double(0x7ff8000000000000LL);
          flag[i] = 3;
          continue;
        }
        if (i == 0 || hist_key(pf, n_faces) != key) atomicAdd(&cnt[key], -(int32_t)i);
        if (i + 1 >= n || hist_key(nf_, n_faces) != key) atomicAdd(&cnt[key], (int32_t)(i + 1));
      }
    }
  }
  if (__any_sync(0xffffffffu, uns) && lane == 0) atomicOr(unsorted, 1);
}

__global__ void k_scatter(int64_t n, const int32_t *__restrict__ face_id, int32_t n_faces,
                          const int32_t *__restrict__ off, int32_t *__restrict__ cursor,
                          const int32_t *__restrict__ unsorted, int32_t *__restrict__ perm) {
  if (!*unsorted) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i - threadIdx.x < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const bool in = i < n;
    const int f = in ? face_id[i] : -1;
    const bool ok = in && f >= 0 && f < n_faces;
    const int key = ok ? f : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    const int leader = __ffs(peers) - 1;
    int base = 0;
    if (ok && (int)(threadIdx.x & 31) == leader) base = atomicAdd(&cursor[f], __popc(peers));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (ok) perm[off[f] + base + __popc(peers & ((1u << (threadIdx.x & 31)) - 1u))] = (int32_t)i;
  }
}

__global__ void k_ntiles(int32_t n_faces, int32_t qu, const int32_t *__restrict__ order,
                         const int32_t *__restrict__ cnt, int32_t *__restrict__ nt) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n_faces) nt[j] = (cnt[order[j]] + qu - 1) / qu;
  if (j == n_faces) nt[j] = 0;
}

__global__ void k_tiles(int32_t n_faces, int32_t max_tiles, int32_t qu, const int32_t *__restrict__ order,
                        const int32_t *__restrict__ cnt, const int32_t *__restrict__ off,
                        const int32_t *__restrict__ toff, Tile *__restrict__ tiles, int32_t *__restrict__ ntiles) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int total = toff[n_faces];
  if (i == 0) *ntiles = total;
  if (i >= total || i >= max_tiles) return;
  int lo = 0, hi = n_faces - 1;                    // last j with toff[j] <= i
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (toff[mid] <= i) lo = mid; else hi = mid - 1;
  }
  const int f = order[lo];
  const int k = i - toff[lo];
  Tile T;
  T.face = f;
  T.qbeg = off[f] + (int64_t)k * qu;
  T.qcnt = min(qu, cnt[f] - k * qu);
  tiles[i] = T;
}

// Implicit-grid batches (wn_query_grid): units are cut per grid, largest
// faces first; no bucketing (a grid is one face's contiguous query range).
__global__ void k_grid_keys(int32_t n_grid, const int32_t *__restrict__ grid_face, int32_t n_faces,
                            const int32_t *__restrict__ face_rec_off, uint32_t *__restrict__ key,
                            int32_t *__restrict__ val) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n_grid) return;
  const int f = grid_face[g];
  const int nrec = (f >= 0 && f < n_faces) ? face_rec_off[f + 1] - face_rec_off[f] : 0;
  key[g] = 0xffffffffu - (uint32_t)nrec;     // ascending key = descending record count
  val[g] = g;
}

__global__ void k_grid_tiles(int32_t n_grid, int32_t tpg, int32_t qu, int64_t G, const int32_t *__restrict__ order,
                             const int32_t *__restrict__ grid_face, int32_t n_faces, Tile *__restrict__ tiles,
                             int32_t *__restrict__ ntiles) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)n_grid * tpg;
  if (i == 0) *ntiles = (int32_t)total;
  if (i >= total) return;
  const int g = order[i / tpg];
  const int k = (int)(i % tpg);
  const int f = grid_face[g];
  Tile T;
  T.face = (f >= 0 && f < n_faces) ? f : -1;
  T.qbeg = (int64_t)g * G + (int64_t)k * qu;
  const int64_t rem = G - (int64_t)k * qu;
  T.qcnt = (int32_t)(rem < qu ? rem : qu);
  tiles[i] = T;
}

static thread_local int32_t g_launches = 0;

// A/B switch (environment): WN_FINISH_Q=0 classifies by scanning the flag array
static bool env_on(const char *name) {
  const char *e = std::getenv(name);
  return !(e && *e && atoi(e) == 0);
}
static bool finish_by_queue() { return env_on("WN_FINISH_Q"); }

// K3 (phase 1, hard pairs, overflow, finish) on prepared tiles
template <typename R>
static wn_status_t launch_k3(wn_faces_t F, const QParams<R> &P, int64_t n, const int32_t *face_id, int max_tiles,
                             cudaStream_t st, int &launches) {
  cudaEvent_t e0 = nullptr, e1 = nullptr, em = nullptr;
  if (F->timing_on) {
    WN_CUDA(cudaEventCreate(&e0));
    WN_CUDA(cudaEventCreate(&em));
    WN_CUDA(cudaEventCreate(&e1));
    WN_CUDA(cudaEventRecord(e0, st));
  }
  const int hb = 148 * WN_HARD_BPS;   // k_hard CTAs (one wave at 4 resident CTAs / SM)
  const bool ang = F->opt.angle_mode == 1;
  const bool grid = P.grid_box != nullptr;
  auto phase1 = [&](auto cnt_tag) {
    constexpr bool C_ = decltype(cnt_tag)::value;
    if (ang) {
      if (grid) k_phase1<R, C_, true, true><<<max_tiles, NTH, 0, st>>>(P);
      else k_phase1<R, C_, true, false><<<max_tiles, NTH, 0, st>>>(P);
    } else {
      if (grid) k_phase1<R, C_, false, true><<<max_tiles, NTH, 0, st>>>(P);
      else k_phase1<R, C_, false, false><<<max_tiles, NTH, 0, st>>>(P);
    }
  };
  if (F->counters_on) {
    WN_CUDA(cudaMemsetAsync(F->counters, 0, 16 * sizeof(unsigned long long), st));
    phase1(std::true_type{});
    if (em) WN_CUDA(cudaEventRecord(em, st));
    k_hard<R, true><<<hb, 256, 0, st>>>(P);
    k_overflow<R><<<148 * 4, 128, 0, st>>>(P, face_id, n);
    k_finish<<<148 * 8, 256, 0, st>>>(n, P.winding, P.flag, P.rule, F->counters);   // (counts the on-boundary queries)
  } else {
    phase1(std::false_type{});
    if (em) WN_CUDA(cudaEventRecord(em, st));
    k_hard<R, false><<<hb, 256, 0, st>>>(P);
    k_overflow<R><<<148 * 4, 128, 0, st>>>(P, face_id, n);
    if (finish_by_queue()) k_finish_q<<<148 * 8, 256, 0, st>>>(P.hq, P.hq_count, P.hq_cap, P.winding, P.flag, P.rule);
    else k_finish<<<148 * 8, 256, 0, st>>>(n, P.winding, P.flag, P.rule, nullptr);
  }
  launches += 4;
  if (F->timing_on) {
    WN_CUDA(cudaEventRecord(e1, st));
    F->k3_events.push_back({e0, e1});
    F->k3_mid.push_back(em);
  }
  WN_CUDA(cudaGetLastError());
  return WN_OK;
}

template <typename R>
static wn_status_t launch_query(wn_faces_t F, int64_t n, const int32_t *face_id, const double *uv,
                                double *winding, uint8_t *flag, cudaStream_t st) {
  const int nf = F->n_faces;
  // unit = up to qu queries of one face per CTA (QT at a time): large batches
  // amortise the CTA prologue and the record staging over several sub-tiles,
  // small ones keep >= ~4 waves of CTAs
  int sub = (int)std::min<int64_t>(16, std::max<int64_t>(1, n / ((int64_t)QT * 148 * 16)));
  if (const char *s = std::getenv("WN_SUBTILES")) sub = std::max(1, std::min(16, atoi(s)));   // <= 16: a unit <= 4096 queries (12-bit rank in the regrouping key)
  const int qu = (QT * sub + QTK - 1) / QTK * QTK;   // whole k_phase1 sub-tiles, <= 4096
  const int64_t max_tiles64 = (n + qu - 1) / qu + nf;
  if (n > INT32_MAX - 1 || max_tiles64 > INT32_MAX) {
    set_error("wn_query: batch too large (n=%lld); split it", (long long)n);
    return WN_ERR_ARG;
  }
  const int max_tiles = (int)max_tiles64;
  int hq_cap = (int)std::min<int64_t>(std::max<int64_t>(n / 8, 1 << 20), 1 << 26);
  if (const char *cap = std::getenv("WN_HQ_CAP")) hq_cap = std::max(1, atoi(cap));   // tests: force overflow
  size_t tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, (int32_t *)nullptr, (int32_t *)nullptr, nf + 1, st);
  size_t need = 0;
  auto carve = [&](size_t bytes) { size_t o = need; need += (bytes + 255) & ~(size_t)255; return o; };
  const size_t o_cnt = carve(sizeof(int32_t) * (nf + 1));
  const size_t o_off = carve(sizeof(int32_t) * (nf + 1));
  const size_t o_cur = carve(sizeof(int32_t) * (nf + 1));
  const size_t o_flags = carve(sizeof(int32_t) * 8);
  const size_t o_nt = carve(sizeof(int32_t) * (nf + 1));
  const size_t o_toff = carve(sizeof(int32_t) * (nf + 1));
  const size_t o_tiles = carve(sizeof(Tile) * (size_t)max_tiles);
  const size_t o_perm = carve(sizeof(int32_t) * (size_t)n);
  const size_t o_sord = carve(sizeof(int32_t) * (size_t)n);
  const size_t o_skey = carve(sizeof(int32_t) * (size_t)n);
  const size_t o_hq = carve(sizeof(HardEntry) * (size_t)hq_cap);
  const size_t o_tmp = carve(tmp);
  char *base = nullptr;
  WN_CUDA(cache_alloc((void **)&base, need, st));
  int32_t *cnt = (int32_t *)(base + o_cnt), *off = (int32_t *)(base + o_off);
  int32_t *cur = (int32_t *)(base + o_cur), *nt = (int32_t *)(base + o_nt);
  int32_t *toff = (int32_t *)(base + o_toff), *flags = (int32_t *)(base + o_flags);
  Tile *tiles = (Tile *)(base + o_tiles);
  int32_t *perm = (int32_t *)(base + o_perm);
  HardEntry *hq = (HardEntry *)(base + o_hq);
  void *tmpb = base + o_tmp;
  int launches = 0;
  // cnt, off, cursor and flags are contiguous at the front: one clear
  WN_CUDA(cudaMemsetAsync(base, 0, o_nt, st));
  const int TB = 256;
  const int64_t nb64 = (n + TB - 1) / TB;
  const int nb = (int)(nb64 < 148 * 32 ? nb64 : 148 * 32);
  const int64_t nbh64 = ((n + 15) / 16 + TB - 1) / TB;
  const int nbh = (int)(nbh64 < 148 * 16 ? nbh64 : 148 * 16);
  k_hist<<<nbh, TB, 0, st>>>(n, face_id, nf, cnt, flags, winding, flag);
  ++launches;
  cub::DeviceScan::ExclusiveSum(tmpb, tmp, cnt, off, nf + 1, st);
  launches += 2;
  k_scatter<<<nb, TB, 0, st>>>(n, face_id, nf, off, cur, flags, perm);
  ++launches;
  k_ntiles<<<(nf + 1 + TB - 1) / TB, TB, 0, st>>>(nf, qu, F->face_order, cnt, nt);
  ++launches;
  cub::DeviceScan::ExclusiveSum(tmpb, tmp, nt, toff, nf + 1, st);
  launches += 2;
  k_tiles<<<(max_tiles + TB - 1) / TB, TB, 0, st>>>(nf, max_tiles, qu, F->face_order, cnt, off, toff, tiles,
                                                   flags + 1);
  ++launches;
  QParams<R> P;
  P.hot = (const Hot<R> *)F->hot;
  P.cold = (const BaseCold<R> *)F->cold;
  P.copy = F->copy;
  P.nq = n;
  P.n_copy = (int32_t)F->n_seg;
  P.n_base = F->n_base;
  P.n_rec = (int32_t)F->n_records;
  P.face_rec_off = F->face_rec_off;
  P.face_cold_off = F->face_cold_off;
  P.face_dom = F->face_dom;
  P.face_per = F->face_per;
  P.face_M = F->face_M;
  P.uv = uv;
  P.winding = winding;
  P.flag = flag;
  P.tiles = tiles;
  P.ntiles = flags + 1;
  P.perm = perm;
  P.unsorted = flags;
  P.hq = hq;
  P.hq_count = flags + 2;
  P.hq_next = flags + 3;
  P.hq_cap = hq_cap;
  P.eps = F->eps;
  P.max_depth = F->max_depth;
  P.rule = F->opt.rule;
  P.counters = F->counters;
  P.grid_box = nullptr;
  P.grid_face = nullptr;
  P.grid_n = 0;
  P.grid_nu = P.grid_nv = 0;
  P.grid_blk = 0;
  P.face_box = F->face_box;
  P.spatial = (F->face_box != nullptr && !(std::getenv("WN_NO_SPATIAL") && *std::getenv("WN_NO_SPATIAL"))) ? 1 : 0;
  P.sorder = (int32_t *)(base + o_sord);
  P.skey = (int32_t *)(base + o_skey);
  {
    const wn_status_t rc = launch_k3<R>(F, P, n, face_id, max_tiles, st, launches);
    if (rc != WN_OK) return rc;
  }
  WN_CUDA(cudaGetLastError());
  cache_free(base, st);
  if (F->last_use) WN_CUDA(cudaEventRecord(F->last_use, st));
  g_launches = launches;
  return WN_OK;
}

template <typename R>
static wn_status_t launch_query_grid(wn_faces_t F, int32_t n_grid, const int32_t *grid_face, const double *grid_box,
                                     int32_t nu, int32_t nv, double *winding, uint8_t *flag, cudaStream_t st) {
  const int nf = F->n_faces;
  const int64_t G = (int64_t)nu * nv;
  const int64_t n = G * n_grid;
  if (n > INT32_MAX - 1) {
    set_error("wn_query_grid: batch too large (%lld queries); split it", (long long)n);
    return WN_ERR_ARG;
  }
  int sub = (int)std::min<int64_t>(16, std::max<int64_t>(1, n / ((int64_t)QT * 148 * 16)));
  if (const char *s = std::getenv("WN_SUBTILES")) sub = std::max(1, std::min(16, atoi(s)));   // <= 16: a unit <= 4096 queries (12-bit rank in the regrouping key)
  const int qu = (QT * sub + QTK - 1) / QTK * QTK;   // whole k_phase1 sub-tiles, <= 4096
  const int tpg = (int)((G + qu - 1) / qu);
  const int64_t max_tiles64 = (int64_t)n_grid * tpg;
  if (max_tiles64 > INT32_MAX) { set_error("wn_query_grid: too many tiles"); return WN_ERR_ARG; }
  const int max_tiles = (int)max_tiles64;
  int hq_cap = (int)std::min<int64_t>(std::max<int64_t>(n / 8, 1 << 20), 1 << 26);
  if (const char *cap = std::getenv("WN_HQ_CAP")) hq_cap = std::max(1, atoi(cap));
  size_t tmp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp, (const uint32_t *)nullptr, (uint32_t *)nullptr,
                                  (const int32_t *)nullptr, (int32_t *)nullptr, n_grid, 0, 32, st);
  size_t need = 0;
  auto carve = [&](size_t bytes) { size_t o = need; need += (bytes + 255) & ~(size_t)255; return o; };
  const size_t o_flags = carve(sizeof(int32_t) * 8);
  const size_t o_k0 = carve(sizeof(uint32_t) * n_grid), o_k1 = carve(sizeof(uint32_t) * n_grid);
  const size_t o_v0 = carve(sizeof(int32_t) * n_grid), o_v1 = carve(sizeof(int32_t) * n_grid);
  const size_t o_tiles = carve(sizeof(Tile) * (size_t)max_tiles);
  const size_t o_hq = carve(sizeof(HardEntry) * (size_t)hq_cap);
  const size_t o_tmp = carve(tmp);
  char *base = nullptr;
  WN_CUDA(cache_alloc((void **)&base, need, st));
  int32_t *flags = (int32_t *)(base + o_flags);
  uint32_t *k0 = (uint32_t *)(base + o_k0), *k1 = (uint32_t *)(base + o_k1);
  int32_t *v0 = (int32_t *)(base + o_v0), *v1 = (int32_t *)(base + o_v1);
  Tile *tiles = (Tile *)(base + o_tiles);
  int launches = 0;
  WN_CUDA(cudaMemsetAsync(flags, 0, sizeof(int32_t) * 8, st));
  const int TB = 256;
  k_grid_keys<<<(n_grid + TB - 1) / TB, TB, 0, st>>>(n_grid, grid_face, nf, F->face_rec_off, k0, v0);
  ++launches;
  cub::DeviceRadixSort::SortPairs(base + o_tmp, tmp, k0, k1, v0, v1, n_grid, 0, 32, st);
  launches += 4;
  k_grid_tiles<<<(max_tiles + TB - 1) / TB, TB, 0, st>>>(n_grid, tpg, qu, G, v1, grid_face, nf, tiles, flags + 1);
  ++launches;
  QParams<R> P;
  P.hot = (const Hot<R> *)F->hot;
  P.cold = (const BaseCold<R> *)F->cold;
  P.copy = F->copy;
  P.nq = n;
  P.n_copy = (int32_t)F->n_seg;
  P.n_base = F->n_base;
  P.n_rec = (int32_t)F->n_records;
  P.face_rec_off = F->face_rec_off;
  P.face_cold_off = F->face_cold_off;
  P.face_dom = F->face_dom;
  P.face_per = F->face_per;
  P.face_M = F->face_M;
  P.uv = nullptr;
  P.winding = winding;
  P.flag = flag;
  P.tiles = tiles;
  P.ntiles = flags + 1;
  P.perm = nullptr;
  P.unsorted = flags;            // 0: the query index is the position
  P.hq = (HardEntry *)(base + o_hq);
  P.hq_count = flags + 2;
  P.hq_next = flags + 3;
  P.hq_cap = hq_cap;
  P.eps = F->eps;
  P.max_depth = F->max_depth;
  P.rule = F->opt.rule;
  P.counters = F->counters;
  P.grid_box = reinterpret_cast<const double2 *>(grid_box);
  P.grid_face = grid_face;
  P.grid_n = G;
  P.grid_nu = nu;
  P.grid_nv = nv;
  P.face_box = F->face_box;
  P.spatial = 0;
  P.sorder = nullptr;
  P.skey = nullptr;
  // 2-D warp blocks when a sub-tile is R whole rows (R = QT / nu) and a block
  // of R rows x (32 / R) columns fits: units start at multiples of QT
  P.grid_blk = 0;
  if (nu > 0 && nu <= QTK && QTK % nu == 0 && QTK / nu <= 32 * QPL &&
      !(std::getenv("WN_GRID_LINEAR") && *std::getenv("WN_GRID_LINEAR")))
    P.grid_blk = 32 * QPL / (QTK / nu);
  {
    const wn_status_t rc = launch_k3<R>(F, P, n, nullptr, max_tiles, st, launches);
    if (rc != WN_OK) return rc;
  }
  WN_CUDA(cudaGetLastError());
  cache_free(base, st);
  if (F->last_use) WN_CUDA(cudaEventRecord(F->last_use, st));
  g_launches = launches;
  return WN_OK;
}

}  // namespace wn

namespace wn {
// Keep stream-ordered allocations cached across synchronisations (the query
// scratch and the records are reallocated every call otherwise).
void ensure_pool(int dev) {
  static int done[64] = {0};
  if (dev < 0 || dev >= 64 || done[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done[dev] = 1;
}
}  // namespace wn

extern "C" wn_status_t wn_query(wn_faces_t faces, int64_t n, const int32_t *face_id, const double *uv,
                                double *winding, uint8_t *flag, void *stream) {
  if (!faces) { wn::set_error("wn_query: NULL handle"); return WN_ERR_ARG; }
  if (n < 0) { wn::set_error("wn_query: n < 0"); return WN_ERR_ARG; }
  if (n == 0) { wn::g_launches = 0; return WN_OK; }
  if (!face_id || !uv || !winding || !flag) { wn::set_error("wn_query: NULL array"); return WN_ERR_ARG; }
  cudaStream_t st = (cudaStream_t)stream;
  WN_CUDA(cudaSetDevice(faces->device));
  wn::ensure_pool(faces->device);
  if (faces->n_faces == 0) {
    // every query references a non-existent face
    wn::set_error("");
  }
  // the build's record emission may still be running on its own stream
  if (faces->ready) WN_CUDA(cudaStreamWaitEvent(st, faces->ready, 0));
  if (faces->precision == 1) return wn::launch_query<float>(faces, n, face_id, uv, winding, flag, st);
  return wn::launch_query<double>(faces, n, face_id, uv, winding, flag, st);
}

extern "C" wn_status_t wn_query_grid(wn_faces_t faces, int32_t n_grid, const int32_t *grid_face,
                                     const double *grid_box, int32_t nu, int32_t nv, double *winding, uint8_t *flag,
                                     void *stream) {
  if (!faces) { wn::set_error("wn_query_grid: NULL handle"); return WN_ERR_ARG; }
  if (n_grid < 0 || nu < 0 || nv < 0) { wn::set_error("wn_query_grid: negative size"); return WN_ERR_ARG; }
  if (n_grid == 0 || nu == 0 || nv == 0) { wn::g_launches = 0; return WN_OK; }
  if (!grid_face || !grid_box || !winding || !flag) { wn::set_error("wn_query_grid: NULL array"); return WN_ERR_ARG; }
  if (((uintptr_t)grid_box & 15) != 0) { wn::set_error("wn_query_grid: grid_box must be 16-B aligned"); return WN_ERR_ARG; }
  cudaStream_t st = (cudaStream_t)stream;
  WN_CUDA(cudaSetDevice(faces->device));
  wn::ensure_pool(faces->device);
  if (faces->ready) WN_CUDA(cudaStreamWaitEvent(st, faces->ready, 0));
  if (faces->precision == 1)
    return wn::launch_query_grid<float>(faces, n_grid, grid_face, grid_box, nu, nv, winding, flag, st);
  return wn::launch_query_grid<double>(faces, n_grid, grid_face, grid_box, nu, nv, winding, flag, st);
}

extern "C" int32_t wn_last_query_launches(void) { return wn::g_launches; }

// Streamed query from HOST buffers: chunks of the batch go host->device on a
// copy-in stream, through wn_query on `stream`, and back on a copy-out stream,
// three chunk slots deep, so the PCIe transfers in both directions overlap the
// kernels of the neighbouring chunks.  Face-sorted input stays face-sorted per
// chunk (K4 then skips its scatter).
extern "C" wn_status_t wn_query_host(wn_faces_t faces, int64_t n, const int32_t *h_face_id, const double *h_uv,
                                     double *h_winding, uint8_t *h_flag, int64_t chunk, void *stream) {
  using namespace wn;
  if (!faces) { set_error("wn_query_host: NULL handle"); return WN_ERR_ARG; }
  if (n < 0) { set_error("wn_query_host: n < 0"); return WN_ERR_ARG; }
  if (n == 0) { g_launches = 0; return WN_OK; }
  if (!h_face_id || !h_uv || !h_flag) { set_error("wn_query_host: NULL array"); return WN_ERR_ARG; }
  const int dev = faces->device;
  WN_CUDA(cudaSetDevice(dev));
  ensure_pool(dev);
  cudaStream_t st = (cudaStream_t)stream;
  constexpr int NS = 3;
  static std::mutex mu;
  static cudaStream_t s_in[64] = {}, s_out[64] = {};
  static cudaEvent_t ev_in[64][NS], ev_q[64][NS], ev_out[64][NS];
  std::lock_guard<std::mutex> lk(mu);
  if (dev < 0 || dev >= 64) { set_error("device index out of range"); return WN_ERR_ARG; }
  if (!s_in[dev]) {
    WN_CUDA(cudaStreamCreateWithFlags(&s_in[dev], cudaStreamNonBlocking));
    WN_CUDA(cudaStreamCreateWithFlags(&s_out[dev], cudaStreamNonBlocking));
    for (int i = 0; i < NS; ++i) {
      WN_CUDA(cudaEventCreateWithFlags(&ev_in[dev][i], cudaEventDisableTiming));
      WN_CUDA(cudaEventCreateWithFlags(&ev_q[dev][i], cudaEventDisableTiming));
      WN_CUDA(cudaEventCreateWithFlags(&ev_out[dev][i], cudaEventDisableTiming));
    }
  }
  if (chunk <= 0) chunk = std::min<int64_t>(std::max<int64_t>(n / 8, (int64_t)1 << 20), (int64_t)1 << 24);
  chunk = std::min(chunk, n);
  const int64_t nchunks = (n + chunk - 1) / chunk;
  const int nslots = (int)std::min<int64_t>(NS, nchunks);
  // device slots, allocated in the copy-in stream's order (their first use)
  int32_t *d_f[NS] = {};
  double *d_uv[NS] = {}, *d_w[NS] = {};
  uint8_t *d_fl[NS] = {};
  // the copy-in stream must not start before the caller's prior work on `stream`
  WN_CUDA(cudaEventRecord(ev_q[dev][0], st));
  WN_CUDA(cudaStreamWaitEvent(s_in[dev], ev_q[dev][0], 0));
  for (int i = 0; i < nslots; ++i) {
    WN_CUDA(cache_alloc((void **)&d_f[i], sizeof(int32_t) * chunk, s_in[dev]));
    WN_CUDA(cache_alloc((void **)&d_uv[i], sizeof(double) * 2 * chunk, s_in[dev]));
    WN_CUDA(cache_alloc((void **)&d_w[i], sizeof(double) * chunk, s_in[dev]));
    WN_CUDA(cache_alloc((void **)&d_fl[i], chunk, s_in[dev]));
  }
  int launches = 0;
  for (int64_t c = 0; c < nchunks; ++c) {
    const int k = (int)(c % NS);
    const int64_t a = c * chunk, cn = std::min(chunk, n - a);
    if (c >= NS) WN_CUDA(cudaStreamWaitEvent(s_in[dev], ev_out[dev][k], 0));   // slot drained
    WN_CUDA(cudaMemcpyAsync(d_f[k], h_face_id + a, sizeof(int32_t) * cn, cudaMemcpyHostToDevice, s_in[dev]));
    WN_CUDA(cudaMemcpyAsync(d_uv[k], h_uv + 2 * a, sizeof(double) * 2 * cn, cudaMemcpyHostToDevice, s_in[dev]));
    WN_CUDA(cudaEventRecord(ev_in[dev][k], s_in[dev]));
    WN_CUDA(cudaStreamWaitEvent(st, ev_in[dev][k], 0));
    wn_status_t rc = wn_query(faces, cn, d_f[k], d_uv[k], d_w[k], d_fl[k], st);
    if (rc != WN_OK) return rc;
    launches += g_launches;
    WN_CUDA(cudaEventRecord(ev_q[dev][k], st));
    WN_CUDA(cudaStreamWaitEvent(s_out[dev], ev_q[dev][k], 0));
    if (h_winding)   // (NULL: classification only -- the winding numbers stay on the device)
      WN_CUDA(cudaMemcpyAsync(h_winding + a, d_w[k], sizeof(double) * cn, cudaMemcpyDeviceToHost, s_out[dev]));
    WN_CUDA(cudaMemcpyAsync(h_flag + a, d_fl[k], cn, cudaMemcpyDeviceToHost, s_out[dev]));
    WN_CUDA(cudaEventRecord(ev_out[dev][k], s_out[dev]));
  }
  // `stream` completes only after every result reached the host
  for (int i = 0; i < nslots; ++i) WN_CUDA(cudaStreamWaitEvent(st, ev_out[dev][i], 0));
  for (int i = 0; i < nslots; ++i) {
    cache_free(d_f[i], st);
    cache_free(d_uv[i], st);
    cache_free(d_w[i], st);
    cache_free(d_fl[i], st);
  }
  g_launches = launches;
  return WN_OK;
}

extern "C" wn_status_t wn_set_timing(wn_faces_t F, int enable) {
  if (!F) { wn::set_error("wn_set_timing: NULL"); return WN_ERR_ARG; }
  F->timing_on = enable ? 1 : 0;
  return WN_OK;
}

namespace wn {
static std::mutex g_orphan_mu;
static std::vector<K3Timing> g_orphan;
void orphan_timing(std::vector<K3Timing> &&ev) {
  std::lock_guard<std::mutex> lk(g_orphan_mu);
  for (auto &x : ev) g_orphan.push_back(x);
}
}  // namespace wn

extern "C" wn_status_t wn_get_timing(wn_faces_t F, double *ms, double *phase1_ms, int64_t *launches) {
  if (!ms || !launches) { wn::set_error("wn_get_timing: NULL"); return WN_ERR_ARG; }
  std::vector<wn::K3Timing> ev;
  if (F) {
    for (size_t i = 0; i < F->k3_events.size(); ++i) ev.push_back({F->k3_events[i].first, F->k3_mid[i], F->k3_events[i].second});
    F->k3_events.clear();
    F->k3_mid.clear();
  } else {
    std::lock_guard<std::mutex> lk(wn::g_orphan_mu);
    ev.swap(wn::g_orphan);
  }
  double tot = 0.0, p1 = 0.0;
  wn_status_t rc = WN_OK;
  for (auto &x : ev) {
    float t = 0.f, tm = 0.f;
    cudaError_t e = cudaEventSynchronize(x.e1);
    if (e == cudaSuccess) e = cudaEventElapsedTime(&t, x.e0, x.e1);
    if (e == cudaSuccess) e = cudaEventElapsedTime(&tm, x.e0, x.em);
    if (e != cudaSuccess && rc == WN_OK) rc = wn::cuda_fail(e, "wn_get_timing");
    tot += t;
    p1 += tm;
    cudaEventDestroy(x.e0);
    cudaEventDestroy(x.em);
    cudaEventDestroy(x.e1);
  }
  *ms = tot;
  if (phase1_ms) *phase1_ms = p1;
  *launches = (int64_t)ev.size();
  return rc;
}
