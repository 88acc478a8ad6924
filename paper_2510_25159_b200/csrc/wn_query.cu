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
  const Cold<R> *cold;
  const int32_t *face_rec_off;
  const int32_t *face_cold_off;
  const double *face_dom;
  const uint8_t *face_per;
  const double *uv;
  double *winding;
  uint8_t *flag;
  const Tile *tiles;
  const int32_t *ntiles;
  const int32_t *perm;
  const int32_t *unsorted;
  R eps;
  int max_depth;
  int rule;
  unsigned long long *counters;
};

// Counters (optional, COUNT=true): 0 pairs tested, 1 hard pairs, 2 nodes,
// 3 evaluations, 4 leaves, 5 max depth, 6 groups culled (warp-level), 7 on-boundary
template <bool COUNT>
__device__ __forceinline__ void cnt_add(unsigned long long *c, int i, unsigned long long v) {
  if (COUNT && v) atomicAdd(c + i, v);
}

// Rational Bezier point by O(n) Horner in s = t/(1-t) (t <= 1/2) or
// s = (1-t)/t (t > 1/2) on homogeneous coefficients (Table 1).
template <typename R>
__device__ __forceinline__ void eval_point(const Cold<R> *__restrict__ C, int n, R t, R &x, R &y) {
  R X, Y, W;
  if (t <= R(0.5)) {
    R s = t / (R(1) - t);
    X = __ldg(&C->cx[n]); Y = __ldg(&C->cy[n]); W = __ldg(&C->cw[n]);
    for (int j = n - 1; j >= 0; --j) {
      X = X * s + __ldg(&C->cx[j]);
      Y = Y * s + __ldg(&C->cy[j]);
      W = W * s + __ldg(&C->cw[j]);
    }
  } else {
    R s = (R(1) - t) / t;
    X = __ldg(&C->cx[0]); Y = __ldg(&C->cy[0]); W = __ldg(&C->cw[0]);
    for (int j = 1; j <= n; ++j) {
      X = X * s + __ldg(&C->cx[j]);
      Y = Y * s + __ldg(&C->cy[j]);
      W = W * s + __ldg(&C->cw[j]);
    }
  }
  R iw = R(1) / W;
  x = X * iw;
  y = Y * iw;
}

// One hard pair (query q, segment ci) by Alg. 1 with an explicit stack of
// right end points.  The root was found hard in phase 1,
// so it is split immediately.  Results go to shared-memory accumulators.
template <typename R, bool COUNT>
__device__ void hard_pair(const QParams<R> &P, const Cold<R> *__restrict__ cold_face, uint32_t e,
                          const R *s_px, const R *s_py, int *s_xs, double *s_fr, int *s_ob) {
  const int q = e & 0xFF;
  const bool angle = (e >> 8) & 1;
  const Cold<R> *C = cold_face + (e >> 9);
  const R qx = s_px[q], qy = s_py[q];
  const R B = __ldg(&C->B), M = __ldg(&C->M);
  const int n = __ldg(&C->n);
  R stx[MAXD + 1], sty[MAXD + 1];
  int8_t std_[MAXD + 1];
  R Lx = __ldg(&C->f0x) - qx, Ly = __ldg(&C->f0y) - qy;
  R dL = dsqrt(Lx * Lx + Ly * Ly);
  stx[0] = __ldg(&C->f1x) - qx;
  sty[0] = __ldg(&C->f1y) - qy;
  std_[0] = 0;
  int sp = 1;
  R ta = R(0);
  int xsum = 0;
  double fsum = 0.0;
  bool ob = false, root = true;
  unsigned long long nodes = 0, evals = 0, leaves = 0;
  int dmax = 0;
  while (sp > 0) {
    const R rx = stx[sp - 1], ry = sty[sp - 1];
    const int d = std_[sp - 1];
    const R dR = dsqrt(rx * rx + ry * ry);
    bool split;
    ++nodes;
    if (root) {
      split = true;
      root = false;
    } else {
      if (dR < P.eps) { ob = true; break; }                 // Alg. 1 line 1
      const R span = ldexp(B, -d) + M;                      // Eq. 2 + margin (R5)
      split = !(dL + dR > span);                            // Alg. 1 line 3
    }
    if (!split) {                                           // chord substitution
      if (angle) fsum += (double)chord_angle(Lx, Ly, rx, ry);
      else xsum += xcount(Lx, Ly, rx, ry);
      ++leaves;
      Lx = rx; Ly = ry; dL = dR;
      ta += ldexp(R(1), -d);
      --sp;
    } else {
      if (d >= P.max_depth) { ob = true; break; }           // depth cap (R6)
      const R tm = ta + ldexp(R(1), -(d + 1));              // m = (a+b)/2
      R mx, my;
      eval_point(C, n, tm, mx, my);
      ++evals;
      std_[sp - 1] = (int8_t)(d + 1);
      stx[sp] = mx - qx;
      sty[sp] = my - qy;
      std_[sp] = (int8_t)(d + 1);
      ++sp;
      dmax = max(dmax, d + 1);
    }
  }
  if (xsum) atomicAdd(&s_xs[q], xsum);
  if (angle) atomicAdd(&s_fr[q], fsum);
  if (ob) s_ob[q] = 1;
  if (COUNT) {
    cnt_add<COUNT>(P.counters, 2, nodes);
    cnt_add<COUNT>(P.counters, 3, evals);
    cnt_add<COUNT>(P.counters, 4, leaves);
    atomicMax(P.counters + 5, (unsigned long long)dmax);
  }
}

template <typename R>
__device__ __forceinline__ bool group_out(const Hot<R> &h, R px, R py);
template <>
__device__ __forceinline__ bool group_out<double>(const Hot<double> &h, double px, double py) {
  const float2 lo = *reinterpret_cast<const float2 *>(&h.a);
  const float2 hi = *reinterpret_cast<const float2 *>(&h.b);
  return !((double)lo.x <= px && px <= (double)hi.x && (double)lo.y <= py && py <= (double)hi.y);
}
template <>
__device__ __forceinline__ bool group_out<float>(const Hot<float> &h, float px, float py) {
  const __half2 hi = *reinterpret_cast<const __half2 *>(&h.c);
  return !(h.a <= px && px <= __half2float(hi.x) && h.b <= py && py <= __half2float(hi.y));
}

template <typename R, bool COUNT>
__global__ void __launch_bounds__(QT, 4) k_query(QParams<R> P) {
  constexpr int RCH = (sizeof(R) == 8) ? 1024 : 2048;   // records per staged chunk (32 KB)
  __shared__ __align__(128) Hot<R> s_rec[RCH];
  __shared__ uint32_t s_q[NWARP][QW];
  __shared__ int s_qn[NWARP];
  __shared__ R s_px[QT], s_py[QT];
  __shared__ int s_xs[QT];
  __shared__ double s_fr[QT];
  __shared__ int s_ob[QT];
  __shared__ __align__(8) uint64_t s_bar;
  __shared__ int s_head;

  if ((int)blockIdx.x >= *P.ntiles) return;               // uniform: no tile
  const Tile T = P.tiles[blockIdx.x];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int f = T.face;
  bool valid = t < T.qcnt;
  const int32_t pos = T.qbeg + t;
  const int32_t qi = valid ? (*P.unsorted ? P.perm[pos] : pos) : 0;
  R px = R(0), py = R(0);
  if (valid) {
    double u = P.uv[2 * (int64_t)qi], v = P.uv[2 * (int64_t)qi + 1];
    if (!isfinite(u) || !isfinite(v)) {
      P.winding[qi] = __longlong_as_double(0x7ff8000000000000LL);
      P.flag[qi] = 3;
      valid = false;
    } else {
      const uint8_t per = P.face_per[f];
      const double *dom = P.face_dom + 4 * f;
      if (per & 1) u = reduce_coord(u, dom[0], dom[1]);
      if (per & 2) v = reduce_coord(v, dom[2], dom[3]);
      px = (R)u;
      py = (R)v;
    }
  }
  s_px[t] = px;
  s_py[t] = py;
  s_xs[t] = 0;
  s_fr[t] = 0.0;
  s_ob[t] = 0;
  if (t == 0) {
    mbar_init(&s_bar, 1);
    fence_mbar_init();
  }
  __syncthreads();

  const int rec0 = P.face_rec_off[f];
  const int nrec = P.face_rec_off[f + 1] - rec0;
  const Cold<R> *cold_face = P.cold + P.face_cold_off[f];
  const R eps = P.eps;

  // per-lane state (coordinates relative to p)
  R cx = R(0), cy = R(0), cd = R(0);   // previous chain point and its distance
  R ax = R(0), ay = R(0);              // group start A
  int xs = 0, halves = 0;
  double fr = 0.0;
  bool onb = false;
  int skip_end = 0;
  int qn = 0;                          // this warp's queue length (warp-uniform)
  unsigned long long c_pairs = 0, c_hard = 0, c_cull = 0;
  unsigned phase = 0;
  int gr = 0;                          // warp-uniform record cursor

  for (int cb = 0; cb < nrec; cb += RCH) {
    const int cn = min(RCH, nrec - cb);
    if (t == 0) {
      fence_proxy_async_smem();
      mbar_arrive_expect_tx(&s_bar, (unsigned)(cn * sizeof(Hot<R>)));
      tma_bulk_g2s(s_rec, P.hot + rec0 + cb, (unsigned)(cn * sizeof(Hot<R>)), &s_bar);
    }
    while (!mbar_try_wait(&s_bar, phase)) {
    }
    phase ^= 1u;
    const int ce = cb + cn;
    while (gr < ce) {
      const Hot<R> h = s_rec[gr - cb];
      const uint32_t meta = h.meta;
      const uint32_t kind = meta & 0xFu;
      const bool act = valid && gr >= skip_end;
      if (kind == K_SEG) {
        // a4: root eps-test and ellipse test (Alg. 1 lines 1-3, Eq. 1 with R9/R5)
        const R dx = h.a - px, dy = h.b - py;
        const R d = dsqrt(dx * dx + dy * dy);
        bool hard = false;
        if (act) {
          onb |= d < eps;
          if (cd + d > h.c) {                               // pruned: chord (a5)
            if (meta & F_ANGLE) fr += (double)chord_angle(cx, cy, dx, dy);
            else xs += xcount(cx, cy, dx, dy);
          } else {
            hard = !onb;
          }
          if (COUNT) ++c_pairs;
        }
        const unsigned m = __ballot_sync(0xffffffffu, hard);
        if (m) {
          if (hard) {
            const int slot = qn + __popc(m & ((1u << lane) - 1u));
            s_q[warp][slot] = hp_pack(t, (meta & F_ANGLE) ? 1 : 0, (int)(meta >> 8));
          }
          qn += __popc(m);
          if (COUNT) c_hard += hard ? 1 : 0;
          if (qn > QW - 32) {                                 // overflow: warp-local drain
            __syncwarp();
            for (int i = lane; i < qn; i += 32)
              hard_pair<R, COUNT>(P, cold_face, s_q[warp][i], s_px, s_py, s_xs, s_fr, s_ob);
            __syncwarp();
            qn = 0;
          }
        }
        cx = dx; cy = dy; cd = d;
      } else if (kind == K_MOVE || kind == K_MOVEG) {
        const R nx = h.a - px, ny = h.b - py;
        const R nd = dsqrt(nx * nx + ny * ny);
        if (act) {
          onb |= nd < eps;
          if (kind == K_MOVEG && !(meta & F_ANGLE)) {
            // gap chord Z -> A' : -omega(p,Z,A') with its crossing
            const R cr = canon_cross(cx, cy, nx, ny);
            fr -= (double)datan2(cr, cx * nx + cy * ny);
            xs += xcount_exact(cx, cy, nx, ny, cr);
          }
        }
        if (kind == K_MOVE) { ax = nx; ay = ny; }
        cx = nx; cy = ny; cd = nd;
      } else if (kind == K_GROUP) {
        // copy-group / closed-loop cull: p outside the group's box => exactly 0
        const bool out = !act || group_out<R>(h, px, py);
        const int skip = (int)(meta >> 8);
        if (__all_sync(0xffffffffu, out)) {
          gr += skip;
          if (COUNT && lane == 0) ++c_cull;
        } else if (out && act) {
          skip_end = gr + 1 + skip;
        }
      } else if (kind == K_LINE) {
        // omega(p,L) = +-1/2, p on L counts as left (R11)
        const R q = (meta & F_AXISV) ? px : py;
        const bool left = (meta & F_GE) ? (q >= h.a) : (q <= h.a);
        if (act) halves += left ? 1 : -1;
      } else if (kind == K_XCH) {
        if (act) xs -= xcount_exact(ax, ay, cx, cy, canon_cross(ax, ay, cx, cy));
      } else if (kind == K_NCH) {
        if (act) fr -= (double)chord_angle(ax, ay, cx, cy);
      } else if (kind == K_CLOSEG) {
        if (act) {
          const R cr = canon_cross(cx, cy, ax, ay);
          fr -= (double)datan2(cr, cx * ax + cy * ay);
          xs += xcount_exact(cx, cy, ax, ay, cr);
        }
      }
      ++gr;
    }
    __syncthreads();   // all warps done with this chunk before it is overwritten
  }

  // ---- phase 2: drain every warp's hard-pair queue with dynamic fetching ----
  if (lane == 0) s_qn[warp] = qn;
  if (t == 0) s_head = 0;
  __syncthreads();
  int pre[NWARP + 1];
  pre[0] = 0;
#pragma unroll
  for (int w = 0; w < NWARP; ++w) pre[w + 1] = pre[w] + s_qn[w];
  const int total = pre[NWARP];
  if (total > 0) {
    for (;;) {
      const int e = atomicAdd(&s_head, 1);
      if (e >= total) break;
      int w = 0;
#pragma unroll
      for (int k = 1; k < NWARP; ++k) w += (e >= pre[k]) ? 1 : 0;
      hard_pair<R, COUNT>(P, cold_face, s_q[w][e - pre[w]], s_px, s_py, s_xs, s_fr, s_ob);
    }
  }
  __syncthreads();

  // ---- a8: reduce, classify, store ----
  if (valid) {
    const bool ob = onb || s_ob[t];
    double w;
    uint8_t fl;
    if (ob) {
      w = __longlong_as_double(0x7ff8000000000000LL);
      fl = 2;
    } else {
      w = (double)(xs + s_xs[t]) + 0.5 * (double)halves + (fr + s_fr[t]) * (1.0 / TWO_PI);
      const double r = w >= 0.0 ? floor(w + 0.5) : -floor(-w + 0.5);
      fl = (P.rule == 0) ? (fabs(r) >= 1.0) : (r >= 1.0);
    }
    P.winding[qi] = w;
    P.flag[qi] = fl;
    if (COUNT && ob) atomicAdd(P.counters + 7, 1ull);
  }
  if (COUNT) {
    cnt_add<COUNT>(P.counters, 0, c_pairs);
    cnt_add<COUNT>(P.counters, 1, c_hard);
    cnt_add<COUNT>(P.counters, 6, c_cull);
  }
}

// ---------------------------------------------------------------------------
// K4: bucketing by face (a3).  Histogram with warp-aggregated atomics and a
// sortedness flag; scatter only when the batch is not grouped by face.
// ---------------------------------------------------------------------------
__global__ void k_hist(int64_t n, const int32_t *__restrict__ face_id, int32_t n_faces,
                       int32_t *__restrict__ cnt, int32_t *__restrict__ unsorted,
                       double *__restrict__ winding, uint8_t *__restrict__ flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i - threadIdx.x < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const bool in = i < n;
    int f = in ? face_id[i] : -1;
    const bool ok = in && f >= 0 && f < n_faces;
    if (in && !ok) {
      winding[i] = __longlong_as_double(0x7ff8000000000000LL);
      flag[i] = 3;
    }
    if (in && i > 0 && face_id[i - 1] > face_id[i]) atomicOr(unsorted, 1);
    const int key = ok ? f : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    const int leader = __ffs(peers) - 1;
    if (ok && (int)(threadIdx.x & 31) == leader) atomicAdd(&cnt[f], __popc(peers));
  }
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

__global__ void k_ntiles(int32_t n_faces, const int32_t *__restrict__ order, const int32_t *__restrict__ cnt,
                         int32_t *__restrict__ nt) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n_faces) nt[j] = (cnt[order[j]] + QT - 1) / QT;
  if (j == n_faces) nt[j] = 0;
}

__global__ void k_tiles(int32_t n_faces, int32_t max_tiles, const int32_t *__restrict__ order,
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
  T.qbeg = off[f] + k * QT;
  T.qcnt = min(QT, cnt[f] - k * QT);
  tiles[i] = T;
}

static thread_local int32_t g_launches = 0;

template <typename R>
static wn_status_t launch_query(wn_faces_t F, int64_t n, const int32_t *face_id, const double *uv,
                                double *winding, uint8_t *flag, cudaStream_t st) {
  const int nf = F->n_faces;
  const int64_t max_tiles64 = (n + QT - 1) / QT + nf;
  if (max_tiles64 > INT32_MAX) {
    set_error("wn_query: batch too large (n=%lld)", (long long)n);
    return WN_ERR_ARG;
  }
  const int max_tiles = (int)max_tiles64;
  // scratch (stream-ordered)
  size_t tmp1 = 0, tmp2 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp1, (int32_t *)nullptr, (int32_t *)nullptr, nf + 1, st);
  size_t tmp = tmp1 > tmp2 ? tmp1 : tmp2;
  size_t need = 0;
  auto carve = [&](size_t bytes) { size_t o = need; need += (bytes + 255) & ~(size_t)255; return o; };
  const size_t o_cnt = carve(sizeof(int32_t) * (nf + 1));
  const size_t o_off = carve(sizeof(int32_t) * (nf + 1));
  const size_t o_cur = carve(sizeof(int32_t) * (nf + 1));
  const size_t o_nt = carve(sizeof(int32_t) * (nf + 1));
  const size_t o_toff = carve(sizeof(int32_t) * (nf + 1));
  const size_t o_flags = carve(sizeof(int32_t) * 4);
  const size_t o_tiles = carve(sizeof(Tile) * (size_t)max_tiles);
  const size_t o_perm = carve(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  const size_t o_tmp = carve(tmp);
  char *base = nullptr;
  WN_CUDA(cudaMallocAsync((void **)&base, need, st));
  int32_t *cnt = (int32_t *)(base + o_cnt), *off = (int32_t *)(base + o_off);
  int32_t *cur = (int32_t *)(base + o_cur), *nt = (int32_t *)(base + o_nt);
  int32_t *toff = (int32_t *)(base + o_toff), *flags = (int32_t *)(base + o_flags);
  Tile *tiles = (Tile *)(base + o_tiles);
  int32_t *perm = (int32_t *)(base + o_perm);
  void *tmpb = base + o_tmp;
  int launches = 0;
  // cnt, off and cursor are contiguous regions: clear all three + flags
  WN_CUDA(cudaMemsetAsync(base, 0, o_nt, st));
  WN_CUDA(cudaMemsetAsync(flags, 0, sizeof(int32_t) * 4, st));
  const int TB = 256;
  const int64_t nb64 = (n + TB - 1) / TB;
  const int nb = (int)(nb64 < 148 * 32 ? (nb64 > 0 ? nb64 : 1) : 148 * 32);
  k_hist<<<nb, TB, 0, st>>>(n, face_id, nf, cnt, flags, winding, flag);
  ++launches;
  cub::DeviceScan::ExclusiveSum(tmpb, tmp, cnt, off, nf + 1, st);
  launches += 2;
  k_scatter<<<nb, TB, 0, st>>>(n, face_id, nf, off, cur, flags, perm);
  ++launches;
  k_ntiles<<<(nf + 1 + TB - 1) / TB, TB, 0, st>>>(nf, F->face_order, cnt, nt);
  ++launches;
  cub::DeviceScan::ExclusiveSum(tmpb, tmp, nt, toff, nf + 1, st);
  launches += 2;
  k_tiles<<<(max_tiles + TB - 1) / TB, TB, 0, st>>>(nf, max_tiles, F->face_order, cnt, off, toff, tiles,
                                                   flags + 1);
  ++launches;
  QParams<R> P;
  P.hot = (const Hot<R> *)F->hot;
  P.cold = (const Cold<R> *)F->cold;
  P.face_rec_off = F->face_rec_off;
  P.face_cold_off = F->face_cold_off;
  P.face_dom = F->face_dom;
  P.face_per = F->face_per;
  P.uv = uv;
  P.winding = winding;
  P.flag = flag;
  P.tiles = tiles;
  P.ntiles = flags + 1;
  P.perm = perm;
  P.unsorted = flags;
  P.eps = (R)F->eps;
  P.max_depth = F->max_depth;
  P.rule = F->opt.rule;
  P.counters = F->counters;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (F->timing_on) {
    WN_CUDA(cudaEventCreate(&e0));
    WN_CUDA(cudaEventCreate(&e1));
    WN_CUDA(cudaEventRecord(e0, st));
  }
  if (F->counters_on) {
    WN_CUDA(cudaMemsetAsync(F->counters, 0, 8 * sizeof(unsigned long long), st));
    k_query<R, true><<<max_tiles, QT, 0, st>>>(P);
  } else {
    k_query<R, false><<<max_tiles, QT, 0, st>>>(P);
  }
  if (F->timing_on) {
    WN_CUDA(cudaEventRecord(e1, st));
    F->k3_events.push_back({e0, e1});
  }
  ++launches;
  WN_CUDA(cudaGetLastError());
  WN_CUDA(cudaFreeAsync(base, st));
  g_launches = launches;
  return WN_OK;
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
  if (faces->n_faces == 0) {
    // every query references a non-existent face
    wn::set_error("");
  }
  if (faces->precision == 1) return wn::launch_query<float>(faces, n, face_id, uv, winding, flag, st);
  return wn::launch_query<double>(faces, n, face_id, uv, winding, flag, st);
}

extern "C" int32_t wn_last_query_launches(void) { return wn::g_launches; }

extern "C" wn_status_t wn_set_timing(wn_faces_t F, int enable) {
  if (!F) { wn::set_error("wn_set_timing: NULL"); return WN_ERR_ARG; }
  F->timing_on = enable ? 1 : 0;
  return WN_OK;
}

extern "C" wn_status_t wn_get_timing(wn_faces_t F, double *ms, int64_t *launches) {
  if (!F || !ms || !launches) { wn::set_error("wn_get_timing: NULL"); return WN_ERR_ARG; }
  double tot = 0.0;
  for (auto &pr : F->k3_events) {
    WN_CUDA(cudaEventSynchronize(pr.second));
    float t = 0.f;
    WN_CUDA(cudaEventElapsedTime(&t, pr.first, pr.second));
    tot += t;
    cudaEventDestroy(pr.first);
    cudaEventDestroy(pr.second);
  }
  *ms = tot;
  *launches = (int64_t)F->k3_events.size();
  F->k3_events.clear();
  return WN_OK;
}
