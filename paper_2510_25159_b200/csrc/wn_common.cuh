// wn_common.cuh -- record layout, device primitives and the faces handle of
// libwn (B200 / sm_100a).  PAPER.md is cited as P:<line>.
//
// Per face the build emits a flat "record program" (hot records, staged in
// shared memory by the query kernel) plus one cold record per emitted curve
// segment (read only by the recursion of hard pairs).
// "Data layout in HBM".
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>
#include <vector>

#include "../../include/wn.h"

// Device-side invariant checks of the CHECKED build (-DWN_CHECKED, see
// scripts/checked_run.sh): bounds of every shared / global index the kernels
// derive.  A failure prints the condition and traps (the launch fails, the
// caller sees WN_ERR_CUDA).  Compiled out otherwise.
#ifdef WN_CHECKED
#include <cstdio>
#define WN_DCHECK(c)                                                                                   \
  do {                                                                                                 \
    if (!(c)) {                                                                                        \
      printf("WN_DCHECK failed %s:%d block %d thread %d: %s\n", __FILE__, __LINE__, (int)blockIdx.x,   \
             (int)threadIdx.x, #c);                                                                    \
      __trap();                                                                                        \
    }                                                                                                  \
  } while (0)
#else
#define WN_DCHECK(c) \
  do {               \
  } while (0)
#endif

namespace wn {

// ---------------------------------------------------------------------------
// hot record kinds (meta & 0xF) and flag bits (meta bits 4..7); meta >> 8 = aux
// ---------------------------------------------------------------------------
enum : uint32_t {
  K_SEG = 0,     // (a,b) = F1, c = root span S0 (Eq. 1 with R5 margin); aux = face-local cold index
  K_SPAN = 1,    // path-hierarchy node: (x,y) = end of the run, span = sum of its S0; aux = subtree records
  K_MOVE = 3,    // (a,b) = chain start; sets group start A and the previous point
  K_MOVEG = 4,   // (a,b) = next chain start after a gap; crossing mode adds the gap terms
  K_GROUP = 5,   // cull header: box rounded outward (fp64 records: fp32 xmin,ymin,xmax + fp32 ymax in x; fp32: half maxima in c); aux = records to skip
  K_LINE = 6,    // a = line coordinate; omega(p,L) = +-1/2
  K_XCH = 7,     // extended copy closing (crossing mode): -c(A -> Z)
  K_NCH = 8,     // extended copy closing (angle mode): -omega(p, A, Z)  (Eq. 5 chord)
  K_CLOSEG = 9,  // open contractible loop: gap chord Z -> A (crossing mode)
  K_SLINE = 10   // (x,y) = point of a line along v = (p Tu, q Tv), aux = (p, q) as two signed 12-bit
                 // fields: omega(p,L) = +-1/2 for the bands of a general class (Prop. 2)
};
// SEG and SPAN (the records of the inner loop) are kinds 0 and 1: one bit test
// ((meta & 0xE) == 0) selects them, one more (meta & 1) tells them apart
constexpr uint32_t F_ANGLE = 1u << 4;   // literal atan2 chord angles (angle_mode = 1)
constexpr uint32_t F_AXISV = 1u << 5;   // LINE parallel to v: test the u coordinate
constexpr uint32_t F_GE = 1u << 6;      // LINE: left iff q >= c (else q <= c)

// K_SLINE aux: class (p, q) packed in meta bits 8..19 / 20..31
__host__ __device__ __forceinline__ uint32_t sline_meta(int p, int q) {
  return K_SLINE | ((uint32_t)(p & 0xFFF) << 8) | ((uint32_t)(q & 0xFFF) << 20);
}

template <typename R>
struct Hot;
// fp64 records carry an fp32 copy of the point and an fp32 span for the
// conservative single-precision filter of the root ellipse test, plus the exact
// fp64 point used for every decision that affects the value.
template <>
struct __align__(32) Hot<double> {
  float fx, fy, fs;   // fp32 point (nearest) and filter span (rounded up, margins included)
  uint32_t meta;
  double x, y;        // exact point (SEG/MOVE/MOVEG), line coordinate (LINE: x), GROUP: fp32 ymax (up) in x's low word
};
template <>
struct __align__(16) Hot<float> {
  float a, b, c;
  uint32_t meta;
};

// Cold records, read only by the recursion of hard pairs (a6).  Split in two:
//  * BaseCold: one per INPUT segment, written by K1 -- everything that is
//    invariant under the lattice translations of lifting and copy emission:
//    the exact stored end points, the derivative bound (A.1; R29),
//    the Horner-ready homogeneous coefficients c_j = C(n,j) w_j (x_j, y_j, 1)
//    of the STORED (unlifted) curve (O(n) evaluation, Table 1), the
//    8 dyadic piece bounds and piece arc-length bounds.
//  * CopyRec: one per EMITTED segment (a lifted, lattice-translated copy),
//    written by k_emit -- its base segment, target face and the two integer
//    translations (lift shift k_s, copy translate k_g).  The copy's end points
//    are lat(lat(x, k_s, T), k_g, T): the same operations k_emit uses for the
//    hot chain points, so they are bit-identical to them (telescoping).
template <typename R>
struct BaseCold;
// Recursion spans (Eq. 2 with the tightest stored bound covering the node):
//   Bq[q]  bound on the dyadic piece [q/8, (q+1)/8] (t-units): nodes of depth
//          d > 3 lie inside one piece, span = Bq[q] 2^-d;
//   Sp[i]  nodes of depth d = 1..3 are unions of whole pieces: span =
//          min(2^-d max Bq, sum of the pieces' arc-length bounds Lq) (R9),
//          tabulated per node, i = 2^d - 2 + k (no per-node loop in k_hard).
// All incl. the relative margin, fp32 rounded up (still upper bounds).
template <>
struct __align__(16) BaseCold<double> {   // 288 B; coefficient pairs on 16-B boundaries
  double x0, y0, xn, yn;   // exact stored (unlifted) end control points
  double B;                // derivative bound incl. relative margin
  int32_t n, pad;          // degree
  double cx[6], cy[6], cw[6];
  float Bq[8];
  float Sp[14];
  float pad2[2];
};
template <>
struct __align__(16) BaseCold<float> {    // 192 B
  double x0, y0, xn, yn;   // exact stored end points (fp64: the hot fp32 points are rounded from the fp64 lift)
  float B;
  int32_t n;
  float cx[6], cy[6], cw[6];
  float Bq[8];
  float Sp[14];
  float pad[2];
};
struct __align__(8) CopyRec {
  int32_t s;          // base record (BaseCold index of the input segment)
  int32_t face;       // face whose domain holds the periods of the translations
  int32_t ksu, ksv;   // lift shift of the segment (0 on non-periodic axes)
  int32_t ku, kv;     // lattice translate of the copy (0 on non-periodic axes)
};

// K1 output for wn_segment_prep (diagnostics): per input segment, no margins
struct SegPrep {
  double B, S0;
  double Bq[8];
  double Lq[8];   // control-polygon lengths of the 8 dyadic pieces (arc-length bounds)
};

// hard-pair queue entry (shared memory): q (9 bits) | angle (1 bit) | cold local index (22 bits)
__host__ __device__ inline uint32_t hp_pack(int q, int angle, int cold) {
  return (uint32_t)q | ((uint32_t)angle << 9) | ((uint32_t)cold << 10);
}
__host__ __device__ inline int hp_q(uint32_t e) { return (int)(e & 0x1FFu); }
__host__ __device__ inline int hp_angle(uint32_t e) { return (int)((e >> 9) & 1u); }
__host__ __device__ inline int hp_cold(uint32_t e) { return (int)(e >> 10); }

struct Tile {
  int32_t face;
  int32_t qcnt;
  int64_t qbeg;
};

// global hard-pair queue entry (phase 2 runs in its own kernel)
struct HardEntry {
  double px, py;      // reduced query point
  int32_t q;          // query index (output position)
  uint32_t c;         // global copy record index (CopyRec) | angle-mode bit 31
};

// build-plan group (host -> device), 32 B
enum : int32_t { G_LOOP = 0, G_COPY = 1, G_LINE = 2 };
enum : int32_t { PF_CULL = 1, PF_ANGLE = 2, PF_TAIL_CLOSEG = 4, PF_TAIL_XCH = 8, PF_TAIL_NCH = 16, PF_TREE = 32,
                 PF_OMIT_ROOT = 64 };   // closed single-chain loop: no root SPAN (its foci coincide)
struct PlanGroup {
  int32_t kind, flags;
  int32_t loop;
  int32_t ku, kv;       // lattice translate added to the lifted loop
  int32_t rec_off;      // global hot record offset of this group
  int32_t cold_off;     // global cold record offset of its first SEG
  int32_t cold_local;   // face-local index of its first SEG
  int32_t nrec;         // hot records of this group (incl. header)
  int32_t face;         // target face
  double M;             // absolute margin of the target face (R5)
};

// per-loop summary written by the lifting kernel (K2a), read by the planner
struct LoopInfo {
  int32_t cu, cv;       // homology class
  int32_t nbrk;         // junctions that are not bit-continuous after lifting
  int32_t closed;       // last end point == first start point (bitwise)
  int32_t err;          // geometry error in one of its segments
  int32_t nseg;
  double sx, sy;        // lifted start point (beta_0)
  double bb[4];         // lifted control-point box xmin, ymin, xmax, ymax
};

constexpr int NTH = 256;         // threads per query CTA
constexpr int QT = NTH;          // queries per tile (one per thread)
constexpr int NWARP = NTH / 32;
constexpr int QW = 128;          // per-warp hard-pair queue capacity
constexpr int MAXD = 64;         // hard cap of the explicit stack
constexpr double TWO_PI = 6.283185307179586476925286766559;

// ---------------------------------------------------------------------------
// device primitives
// ---------------------------------------------------------------------------
__device__ __forceinline__ double dsqrt(double x) { return sqrt(x); }
__device__ __forceinline__ float dsqrt(float x) { return sqrtf(x); }
__device__ __forceinline__ double datan2(double y, double x) { return atan2(y, x); }
__device__ __forceinline__ float datan2(float y, float x) { return atan2f(y, x); }

// Branch-cut crossing of the chord a -> b (coordinates relative to p) with the
// ray {p + s(-1,0), s >= 0}: the integer c with
//     omega(p,a,b) = (theta(b) - theta(a)) / 2pi + c,
// theta = atan2 in (-pi, pi].  Exact; valid when p
// is not on the chord, which the ellipse margin guarantees for pruned chords.
template <typename R>
__device__ __forceinline__ int xcount(R ax, R ay, R bx, R by) {
  bool ua = ay >= R(0), ub = by >= R(0);
  if (ua == ub) return 0;
  R cr = ax * by - ay * bx;
  return ua ? (cr >= R(0) ? 1 : 0) : (cr < R(0) ? -1 : 0);
}

// Same, for chords p may lie on (gap / copy-closing chords): also covers the
// horizontal chord through p, consistent with omega(p,a,b) = +1/2 there (R11).
// `cr` must be the canonicalised cross product also fed to atan2.
template <typename R>
__device__ __forceinline__ int xcount_exact(R ax, R ay, R bx, R by, R cr) {
  bool ua = ay >= R(0), ub = by >= R(0);
  if (ua && !ub) return cr >= R(0) ? 1 : 0;
  if (!ua && ub) return cr < R(0) ? -1 : 0;
  if (ua && ub && ay == R(0) && by == R(0) && ax < R(0) && bx > R(0)) return 1;
  return 0;
}

template <typename R>
__device__ __forceinline__ R canon_cross(R ax, R ay, R bx, R by) {
  R cr = ax * by - ay * bx;
  return cr == R(0) ? R(0) : cr;   // -0 -> +0 (R11)
}

// Lattice translate x + k T with explicit roundings (no contraction): the one
// formula every lifted / translated point of the library goes through, so
// chain points computed by different kernels are bit-identical.
__device__ __forceinline__ double lat(double x, int k, double T) { return __dadd_rn(x, __dmul_rn((double)k, T)); }

// The frame of an emitted copy (CopyRec): lat(lat(x, k_s, T), k_g, T) =
// (x + k_s T) + k_g T per axis, with the products precomputed (same roundings).
struct CopyFrame {
  double au, bu, av, bv;   // k_s Tu, k_g Tu, k_s Tv, k_g Tv
  __device__ __forceinline__ double X(double x) const { return __dadd_rn(__dadd_rn(x, au), bu); }
  __device__ __forceinline__ double Y(double y) const { return __dadd_rn(__dadd_rn(y, av), bv); }
};
__device__ __forceinline__ CopyFrame copy_frame(const CopyRec &c, const double *__restrict__ face_dom) {
  const double Tu = face_dom[4 * c.face + 1], Tv = face_dom[4 * c.face + 3];
  CopyFrame F;
  F.au = __dmul_rn((double)c.ksu, Tu);
  F.bu = __dmul_rn((double)c.ku, Tu);
  F.av = __dmul_rn((double)c.ksv, Tv);
  F.bv = __dmul_rn((double)c.kv, Tv);
  return F;
}

// omega(p,a,b) * 2pi = atan2(cross, dot) (R7, R11), coordinates relative to p
template <typename R>
__device__ __forceinline__ R chord_angle(R ax, R ay, R bx, R by) {
  R cr = canon_cross(ax, ay, bx, by);
  return datan2(cr, ax * bx + ay * by);
}

}  // namespace wn

// ---------------------------------------------------------------------------
// the faces handle
// ---------------------------------------------------------------------------
struct wn_faces_s {
  int32_t n_faces = 0;
  int precision = 0;
  wn_options_t opt{};
  double eps = 1e-10;
  int max_depth = 48;
  int device = 0;
  void *hot = nullptr;             // Hot<R>[n_records]
  void *cold = nullptr;            // BaseCold<R>[n input segments]
  wn::CopyRec *copy = nullptr;     // [n_seg] emitted segments
  int owns_cold = 1;               // 0: `cold` borrowed from another handle (pairing probes)
  int32_t n_base = 0;              // input segments (BaseCold records)
  int32_t *inv = nullptr;          // [n_base] input segment -> its BaseCold record
  int32_t *face_rec_off = nullptr; // [n_faces+1]
  int32_t *face_cold_off = nullptr;// [n_faces+1]
  int32_t *face_order = nullptr;   // [n_faces] by cost, descending
  double *face_dom = nullptr;      // [n_faces][4]
  uint8_t *face_per = nullptr;     // [n_faces]
  uint8_t *face_ok = nullptr;      // [n_faces]
  double *face_M = nullptr;        // [n_faces] absolute margin M (R5) per face
  float4 *face_box = nullptr;      // [n_faces] box holding every query that can be inside (query regrouping)
  unsigned long long *counters = nullptr;  // [8]
  int counters_on = 0;
  cudaEvent_t last_use = nullptr;    // recorded after the build and after every query
  cudaEvent_t ready = nullptr;       // recorded after the build's record emission
  int timing_on = 0;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> k3_events;
  std::vector<cudaEvent_t> k3_mid;   // after phase 1 (k_phase1) of each timed query
  int64_t n_records = 0, n_seg = 0, n_groups = 0, n_lines = 0, bytes = 0, n_copy_groups = 0, n_bands = 0;
  int32_t max_face_records = 0;
};

namespace wn {
// K3 timing events (begin, after phase 1, end) of handles freed before their
// timing was read: wn_get_timing(NULL, ...) reads them
struct K3Timing { cudaEvent_t e0, em, e1; };
void orphan_timing(std::vector<K3Timing> &&ev);
void ensure_pool(int dev);
cudaError_t cache_alloc(void **out, size_t bytes, cudaStream_t st);
void cache_free(void *p, cudaStream_t st);
void cache_trim();
void set_error(const char *fmt, ...);
wn_status_t cuda_fail(cudaError_t e, const char *what);
}  // namespace wn

#define WN_CUDA(call)                                          \
  do {                                                         \
    cudaError_t e__ = (call);                                  \
    if (e__ != cudaSuccess) return wn::cuda_fail(e__, #call);  \
  } while (0)
