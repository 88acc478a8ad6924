/*
 * wn.h -- C ABI of libwn: batched generalized-winding-number containment
 * queries on trimmed faces, B200 (sm_100a) native.
 *
 * Problem (Sec. 4.1): "Given a test point p and a set of
 * trimming curves {gamma_i} ... determine whether p lies within the trimmed
 * region" by computing the generalized winding number
 *     omega(p) = (1/2pi) * integral over the boundary of d(theta)
 * (Sec. 3.2) and classifying p by it.  Curves are (rational) Bezier
 * p-curves of degree 1..5; faces may be periodic in u and/or v
 * (cylinder / torus, Sec. 4.3-4.5); loops of periodic faces are
 * lifted to the universal covering space.
 *
 * Memory: every array argument is a DEVICE pointer unless marked [host].  The
 * caller owns all input and output buffers; the library owns the faces handle
 * and the records it built.  All GPU work is ordered on the given stream.
 * Errors: functions return wn_status_t; a message for the calling thread is
 * available from wn_last_error() until that thread's next libwn call.  No C++
 * exception crosses this boundary.  Nothing here ever runs on the CPU in place
 * of the GPU: without a usable CUDA device every call fails with WN_ERR_CUDA.
 */
#ifndef WN_H_
#define WN_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct wn_faces_s *wn_faces_t;

typedef enum {
  WN_OK = 0,
  WN_ERR_ARG = 1,       /* NULL pointer, bad count, bad CSR, degree not in 1..5, bad option */
  WN_ERR_GEOM = 2,      /* weight <= 0 or non-finite control point / weight / period */
  WN_ERR_TOPOLOGY = 3,  /* a face violates Prop. 1 / B.1 / B.3 (see face_status) */
  WN_ERR_CUDA = 4,      /* CUDA runtime error or no usable device */
  WN_ERR_NOMEM = 5,     /* device allocation failed */
  WN_ERR_UNSUPPORTED = 6/* valid input outside what this build implements (see face_status) */
} wn_status_t;

/* Per-face validation codes written to face_status by wn_build_faces. */
enum {
  WN_FACE_OK = 0,
  WN_FACE_B1 = 1,          /* |class| > 1 on a uni-periodic axis (Prop. B.1) */
  WN_FACE_UNBALANCED = 2,  /* #A != #B: loops not null-homologous (Prop. 1) */
  WN_FACE_CLASS = 3,       /* mixed classes or gcd(|p|,|q|) != 1 (Props. B.3/B.4) */
  WN_FACE_GENERAL_PQ = 4,  /* (unused: general bi-periodic classes (p,q), Prop. 2, are supported) */
  WN_FACE_PAIRING = 5,     /* PairLoops (Alg. 9) found no proper translate */
  WN_FACE_GEOM = 6         /* bad degree / weight / non-finite data in this face */
};

typedef struct {                 /* [host] */
  double eps;       /* on-boundary tolerance (Alg. 1 line 1) in face parameter units;
                       <= 0 selects the default 1e-10 (fp64) / 1e-6 (fp32)  [reading R1]      */
  int max_depth;    /* explicit-stack depth cap for Alg. 1's recursion (Lemma 2);
                       0 selects 48; must be <= 64  [reading R6]                              */
  int precision;    /* 0 = fp64 records and arithmetic, 1 = fp32 (inputs/outputs stay fp64)   */
  int rule;         /* 0 = nonzero (|round(w)| >= 1, default), 1 = positive (round(w) >= 1)  [R10] */
  int angle_mode;   /* 0 = telescoped branch-cut crossings (default),
                       1 = literal per-chord atan2 (the paper's WindingNumberLineSegment)     */
  int strict;       /* 1 = reject faces violating Prop. 1 (default); 0 = evaluate an
                       unbalanced uni-periodic loop set anyway (single extended curves)        */
  int hierarchy;    /* 1 = path hierarchy over bit-continuous chains (span = sum of
                       the segments' root spans; default), 0 = flat segment list              */
} wn_options_t;

/* Build the per-face records (segment prep K1, lifting K2a, copy emission K2c).
 *   n_faces, n_loops, n_segs >= 0 (n_segs may be 0 only with n_loops == 0).
 *   ctrl_uv       [sum(deg+1)][2] packed control points in STORED (possibly seam-
 *                 discontinuous, reading R18) coordinates; the control points of
 *                 segment s start at the exclusive prefix sum of (deg+1).
 *   ctrl_w        [sum(deg+1)] weights > 0, or NULL for polynomial segments.
 *   seg_degree    [n_segs] in 1..5.
 *   loop_seg_off  [n_loops+1] CSR into segments; segment order = loop orientation
 *                 (interior to the left).
 *   face_loop_off [n_faces+1] CSR into loops.
 *   face_periodic [n_faces] bit0 = periodic in u, bit1 = periodic in v.
 *   face_domain   [n_faces][4] = (u0, Tu, v0, Tv); T used only on periodic axes (R17).
 *   opts          [host] options, or NULL for defaults.
 *   stream        cudaStream_t (0 = legacy default stream).
 *   out           [host] receives the handle on WN_OK; untouched otherwise.
 *   face_status   [n_faces] DEVICE int32 or NULL: WN_FACE_* per face.
 * Synchronisation and input lifetime: the call waits on the host
 * for the device planner's summary (topology validation and the record counts;
 * errors are returned synchronously) and for the segment-prep kernel, the last
 * reader of the caller's arrays -- every later step reads library-owned copies
 * (the lifted control points, CSR copies).  So ALL input buffers may be freed or
 * overwritten, on any stream, as soon as wn_build_faces returns.  The record
 * emission itself stays asynchronous on `stream` after the return; queries may
 * be issued at once on any stream (wn_query waits for the build's event);
 * wn_free_faces orders its frees after the handle's last build/query. */
wn_status_t wn_build_faces(int32_t n_faces, int32_t n_loops, int32_t n_segs, const double *ctrl_uv,
                           const double *ctrl_w, const int32_t *seg_degree,
                           const int32_t *loop_seg_off, const int32_t *face_loop_off,
                           const uint8_t *face_periodic, const double *face_domain,
                           const wn_options_t *opts, void *stream, wn_faces_t *out,
                           int32_t *face_status);

/* NURBS p-curves (p-curves are "(rational) Bezier or NURBS curves"
 * and "B-spline or NURBS curves can always be subdivided into (rational)
 * Bezier segments").  Curve c has degree curve_degree[c] in 1..5, control
 * points ctrl_uv[curve_ctrl_off[c] .. curve_ctrl_off[c+1]) ([.][2] float64),
 * weights ctrl_w (NULL = polynomial B-splines) and the clamped, non-decreasing
 * knot vector knots[curve_knot_off[c] .. curve_knot_off[c+1]) (exactly p+1
 * equal knots at each end) with
 * n_knots(c) = n_ctrl(c) + p + 1 and interior multiplicities <= p.  Every
 * interior knot span of positive length becomes one Bezier segment of the
 * curve's degree; the curve's two end points are copied bit-exactly (the
 * junctions of a loop of curves stay bit-continuous).  All arrays are device
 * pointers; n_ctrl / n_knots are the lengths of ctrl_uv / knots.
 *
 * wn_nurbs_to_bezier: the decomposition alone, into caller buffers in the
 * layout wn_build_faces takes: curve_seg_off [n_curves+1] (segments of curve
 * c = [curve_seg_off[c], curve_seg_off[c+1])), bez_uv [n_pts][2], bez_w
 * [n_pts], bez_degree [n_segs].  seg_cap / pt_cap are their capacities
 * (enough: sum_c (n_ctrl(c) - p_c) segments, sum_c (n_ctrl(c) - p_c)(p_c + 1)
 * points); *n_segs_out / *n_pts_out [host] receive the sizes (also when the
 * capacity is too small: WN_ERR_ARG).  Invalid curve data: WN_ERR_GEOM with
 * the first bad curve in wn_last_error().  Synchronises `stream` once (sizes).
 *
 * wn_build_faces_nurbs: wn_build_faces on NURBS loops: loop l is the curves
 * [loop_curve_off[l], loop_curve_off[l+1]) in order; other arguments and the
 * handle, options, status and error semantics as for wn_build_faces. */
wn_status_t wn_nurbs_to_bezier(int32_t n_curves, int32_t n_ctrl, int32_t n_knots, const double *ctrl_uv,
                               const double *ctrl_w, const int32_t *curve_degree, const int32_t *curve_ctrl_off,
                               const double *knots, const int32_t *curve_knot_off, int32_t seg_cap,
                               int32_t pt_cap, int32_t *curve_seg_off, double *bez_uv, double *bez_w,
                               int32_t *bez_degree, int32_t *n_segs_out, int32_t *n_pts_out, void *stream);

wn_status_t wn_build_faces_nurbs(int32_t n_faces, int32_t n_loops, int32_t n_curves, int32_t n_ctrl,
                                 int32_t n_knots, const double *ctrl_uv, const double *ctrl_w,
                                 const int32_t *curve_degree, const int32_t *curve_ctrl_off, const double *knots,
                                 const int32_t *curve_knot_off, const int32_t *loop_curve_off,
                                 const int32_t *face_loop_off, const uint8_t *face_periodic,
                                 const double *face_domain, const wn_options_t *opts, void *stream,
                                 wn_faces_t *out, int32_t *face_status);

/* Batched query (hot path: bucketing K4 + query kernel K3), fully asynchronous
 * on `stream`; outputs are valid after the stream is synchronised.
 *   n        number of queries (>= 0).
 *   face_id  [n] int32 face index; any order (grouped input skips the sort).
 *   uv       [n][2] float64 query points; periodic coordinates are reduced into
 *            the base tile [u0,u0+T) (kept bit-exact when already inside).
 *   winding  [n] float64 generalized winding number; NaN when flag is 2 or 3.
 *   flag     [n] uint8: 0 outside, 1 inside, 2 on-boundary (within eps of a curve
 *            point visited by Alg. 1, or depth cap), 3 invalid query (bad face_id,
 *            non-finite uv).  Per-query problems never fail the batch.
 * Concurrent calls on one handle from different streams are allowed. */
wn_status_t wn_query(wn_faces_t faces, int64_t n, const int32_t *face_id, const double *uv,
                     double *winding, uint8_t *flag, void *stream);

/* Streamed batched query from HOST buffers (pinned for overlap; pageable works
 * synchronously): the batch is cut into chunks of `chunk` queries (<= 0: auto)
 * that are copied in on an internal copy stream, queried with wn_query on
 * `stream`, and copied back on a second copy stream, three chunks deep, so
 * host<->device transfers in both directions overlap the kernels.  Arguments
 * as for wn_query, but h_* are host pointers owned by the caller that must stay
 * valid until `stream` is synchronised; the results are in h_winding / h_flag
 * once it is.  Same per-query semantics as wn_query.  h_winding may be NULL:
 * only the classification (the containment answer) is copied back,
 * 1 B per query instead of 9. */
wn_status_t wn_query_host(wn_faces_t faces, int64_t n, const int32_t *h_face_id, const double *h_uv,
                          double *h_winding, uint8_t *h_flag, int64_t chunk, void *stream);

/* Implicit-grid query: the tessellation application of Sec. 5.4.3 (P:884-895:
 * "sample a uniform grid in the parametric domain", then classify) and the
 * paper's per-shape 256x256 sample grids.  Grid g queries the nu x nv
 * cell centres of the box grid_box[g] of face grid_face[g]; no uv is read from
 * memory (0 B/query in), only the results are written.
 *   n_grid     number of grids (>= 0); grid_face [n_grid] int32 (device).
 *   grid_box   [n_grid][4] float64 (device, 16-B aligned) = (u_lo, v_lo, u_hi, v_hi).
 *   nu, nv     cells per grid along u and v (>= 0); n_grid * nu * nv < 2^31.
 *   winding, flag  [n_grid][nv][nu] (row-major: v outer, u inner), semantics
 *            as for wn_query.  Query (g, iv, iu) is the point
 *              u = u_lo + (iu + 0.5) * ((u_hi - u_lo) / nu),
 *              v = v_lo + (iv + 0.5) * ((v_hi - v_lo) / nv),
 *            each operation rounded in this order (no contraction), so an
 *            explicit batch built by the same formula gives identical points.
 *   An invalid grid_face sets flag 3 for the grid's queries; a non-finite box
 *   gives non-finite points (flag 3).  Asynchronous on `stream` like wn_query. */
wn_status_t wn_query_grid(wn_faces_t faces, int32_t n_grid, const int32_t *grid_face, const double *grid_box,
                          int32_t nu, int32_t nv, double *winding, uint8_t *flag, void *stream);

typedef struct {
  int64_t n_records;     /* hot records (MOVE/SEG/GROUP/LINE/...) over all faces */
  int64_t n_seg_records; /* SEG records (input segments x emitted lattice copies) */
  int64_t n_groups;      /* cullable groups (closed loops and extended copies) */
  int64_t n_lines;       /* LINE records (Eq. 5 / Eq. 8 line terms) */
  int64_t bytes;         /* device bytes owned by the handle */
  int32_t precision;     /* 0 fp64, 1 fp32 */
  int32_t max_face_records;
  int64_t n_copy_groups; /* extended-copy groups (Eq. 5 copies of non-contractible loops) */
  int64_t n_bands;       /* Eq. 8 bands emitted for bi-periodic pairs: line pairs */
} wn_faces_info_t;

wn_status_t wn_faces_info(wn_faces_t faces, wn_faces_info_t *out /* [host] */);

/* Device-side event counters of the last wn_query on this handle, enabled by
 * wn_set_counters(faces, 1) (adds atomics; for diagnostics, not for timing).
 * out[host][12] = {root (query, segment) tests, hard pairs, recursion nodes,
 *                  split-point evaluations, leaves, max depth, warp-level skips
 *                  (culled groups + pruned hierarchy subtrees), on-boundary,
 *                  (query, hierarchy node) tests, phase-1 warp-record
 *                  iterations, hierarchy-node tests that descend (the others
 *                  substitute the run's chord), segment tests that substitute
 *                  the chord}. */
wn_status_t wn_set_counters(wn_faces_t faces, int enable);
wn_status_t wn_get_counters(wn_faces_t faces, void *stream, int64_t *out /* [host][12] */);

/* In-library timing of the query kernel K3 (CUDA events recorded on the
 * launching stream around every K3 launch -- phase 1, hard pairs, overflow,
 * finish -- and after its phase 1, while enabled).  wn_get_timing waits for the
 * recorded events, returns the summed K3 and phase-1 milliseconds and the
 * number of timed queries since the last call, and resets them.  faces = NULL
 * reads the timing of handles that were freed before it was read. */
wn_status_t wn_set_timing(wn_faces_t faces, int enable);
wn_status_t wn_get_timing(wn_faces_t faces, double *k3_ms /* [host] */, double *phase1_ms /* [host] or NULL */,
                          int64_t *k3_launches /* [host] */);

/* K1 segment prep on its own (diagnostics / tests): for every segment writes
 * out[s][18] = {B, S0, Bq[0..7], Lq[0..7]}: the derivative bound of Lemma 1
 * (App. A.1, reading R29), the root span S0 = min(B,
 * control-polygon length, sum of Lq) (R9), the derivative bounds of the 8
 * dyadic pieces [q/8,(q+1)/8] (t-units) and their control-polygon lengths
 * (arc-length bounds), without margins.  Device pointers; synchronises the
 * stream. */
wn_status_t wn_segment_prep(int32_t n_segs, const double *ctrl_uv, const double *ctrl_w,
                            const int32_t *seg_degree, double *out, void *stream);

/* Diagnostics: the device's measured FMA pipe peak (the roofline denominator of
 * the query kernel): dependent-FMA chains, 8 independent per
 * thread, 4 CTAs of 256 threads per SM, launches of ~`seconds` each, best of
 * three.  fp32 = 0: DFMA, 1: FFMA.  *lane_fma_per_s [host] = lane FMA
 * instructions per second (FLOP/s = 2x); *sm_mhz [host, or NULL] = the SM
 * clock during the best launch (clock64 cycles / globaltimer ns of CTA 0).
 * Synchronous; uses the current device. */
wn_status_t wn_measure_fp_peak(int fp32, double seconds, double *lane_fma_per_s, double *sm_mhz);

/* Diagnostics: the recursion bounds the handle's hard-pair recursion uses, per
 * INPUT segment s (in wn_build_faces order): out[s][23] = {B, Bq[0..7],
 * Sp[0..13]} -- the derivative bound of Lemma 1 / App. A.1 (P:335-345,
 * P:1095-1109, R29) with its relative margin, the bounds of the 8 dyadic
 * pieces [q/8,(q+1)/8] (used for nodes of depth > 3, span = Bq 2^-d, Eq. 2
 * P:351-356) and the spans of the depth-1..3 nodes (index 2^d - 2 + k: the
 * minimum of 2^-d max Bq and the pieces' arc-length bounds, R9), as stored
 * (fp32, rounded up).  `out` is a device pointer; synchronises `stream`. */
wn_status_t wn_recursion_bounds(wn_faces_t faces, double *out, void *stream);

/* libwn keeps freed device buffers (records, query scratch) in a per-device
 * cache for reuse; wn_trim_memory returns them to the driver. */
void wn_trim_memory(void);

/* Release the handle; the caller guarantees no query on it is in flight. */
void wn_free_faces(wn_faces_t faces);

/* Thread-local message for the last failing call on this thread ("" if none). */
const char *wn_last_error(void);

/* Number of kernel launches issued by the last wn_query / wn_build_faces on
 * this thread (library kernels only; cub scans count as their kernels). */
int32_t wn_last_query_launches(void);
int32_t wn_last_build_launches(void);

#ifdef __cplusplus
}
#endif
#endif /* WN_H_ */
