/*
 * oracle/wn_oracle.c -- CPU ORACLE.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (its cpu_baseline leg and
 * `--impl reference`) may load or call this library.  The product path
 * (paper_2510_25159_b200/, include/) never does, and shares no code with it.
 *
 * What it computes (PAPER.md = "P:<line>"):
 *   The generalized winding number (GWN) of a trimmed face's boundary loops at
 *   a query point p,  omega(p) = (1/2pi) * integral of d(theta)  (P:246-252,
 *   Sec. 3.2), summed over loops and segments by additivity (Eq. 1).
 *   The paper's ellipse method reaches this exact value faster; the oracle
 *   reaches it by a DIFFERENT exact scheme so the two share nothing:
 *     - each (rational) Bezier segment is subdivided adaptively at t = 1/2 by
 *       homogeneous de Casteljau (the "control-points bound"), and a
 *       piece whose control-point bounding box lies farther than delta from p
 *       is replaced by its chord -- exact by homotopy invariance (P:260-271,
 *       Eq. 3): the piece lies in its convex hull, inside the box, a convex set
 *       not containing p;
 *     - chord winding omega(p,a,b) = atan2(cross, dot)/2pi  (reading R7),
 *       cross == 0 canonicalised to +0 (reading R11);
 *     - long sums use Neumaier compensation.
 *   Periodic faces (Sec. 4.3-4.5):
 *     - own lifting of seam-discontinuous loops to the covering space by the
 *       nearest-translate junction rule (readings R17, R18), homology class by
 *       rounding the closure vector;
 *     - uni-periodic: contractible loops summed over lattice translates
 *       (P:515-516); non-contractible loops by Eq. 5 TAKEN LITERALLY with a
 *       finite N: sum_{k=-N..N} omega(p, gamma + k v) + omega(p,L)
 *       - omega(p, beta_{-N}, beta_{N+1}), omega(p,L) = +-1/2 by the left/right
 *       test (on L counts as left, R11);
 *     - bi-periodic (any coprime class (p,q), Prop. 2): contractible
 *       loops summed over a lattice window; each proper pair (alpha, beta-bar)
 *       by Eq. 8 summed over every band (r,s) -- indexed by the
 *       integer m = p*s - q*r -- in a window, each term an Eq. 5 extended
 *       winding; pairing by the paper's ToLeft / PairLoop / PairLoops (Algs.
 *       7-9) over a transverse window (R16).
 *   Classification: nonzero rule (R10): inside iff |round_half_away(w)| >= 1;
 *   "positive" rule optional.
 *   Distance certificate: dist_lb(p) = min over terminal pieces of the distance
 *   from p to the piece's box (the pieces cover the curve).  A query is
 *   COMPARABLE iff no terminal piece lies within delta and its winding value is
 *   farther than tol from every half-integer.
 *
 * Pins (tests/test_oracle_*.py, -m "not gpu"): SPEC worked values, textbook
 * crossing-number point-in-polygon, exact rational circles, the open-arc closed
 * form, star-shaped analytic classification, the torus-band closed form,
 * Eq. 5 N vs 2N, translation / tile periodicity, gap-closure identity,
 * dense-polyline brute force.  Functions without such a pin say so below.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_TWO_PI 6.283185307179586476925286766559
#define ORC_MAXDEG 5
#define ORC_MAXDEPTH 60

/* ------------------------------------------------------------------------ */
/* Neumaier-compensated accumulator                                          */
/* ------------------------------------------------------------------------ */
typedef struct {
  double s, c;
  double dist_lb;
  int near;
  long pieces;
} acc_t;

static void acc_init(acc_t *A) {
  A->s = 0.0; A->c = 0.0; A->dist_lb = INFINITY; A->near = 0; A->pieces = 0;
}
static void nadd(acc_t *A, double x) {
  double t = A->s + x;
  if (fabs(A->s) >= fabs(x)) A->c += (A->s - t) + x;
  else A->c += (x - t) + A->s;
  A->s = t;
}
static double acc_val(const acc_t *A) { return A->s + A->c; }

/* ------------------------------------------------------------------------ */
/* Primitives                                                               */
/* ------------------------------------------------------------------------ */

/* omega(p, a, b): winding number of the oriented chord a->b about p, from its
 * angular difference.  atan2(cross, dot)/2pi in (-1/2, 1/2]
 * (R7); cross == +-0 canonicalised to +0 so p on the open chord gives +1/2
 * (R11).  PINNED by tests/golden/worked_values.json "chord" (the paper's
 * normalisation P:248-252; SPEC S:158-159 print half these values, reading R26). */
double orc_chord(double px, double py, double ax, double ay, double bx, double by) {
  double ux = ax - px, uy = ay - py, vx = bx - px, vy = by - py;
  double cr = ux * vy - uy * vx;
  double dt = ux * vx + uy * vy;
  if (cr == 0.0) cr = 0.0;
  return atan2(cr, dt) / ORC_TWO_PI;
}

/* Homogeneous control points H[j] = (w_j x_j, w_j y_j, w_j) of a (rational)
 * Bezier segment (rational case App. A.1). */
static void to_hom(int n, const double *P, const double *w, double *H) {
  for (int j = 0; j <= n; j++) {
    double wj = w ? w[j] : 1.0;
    H[3 * j + 0] = wj * P[2 * j + 0];
    H[3 * j + 1] = wj * P[2 * j + 1];
    H[3 * j + 2] = wj;
  }
}

/* de Casteljau split at t = 1/2 in homogeneous coordinates (the subdivision
 * the paper's ellipse bound avoids). */
static void hsplit(int n, const double *H, double *L, double *R) {
  double tmp[(ORC_MAXDEG + 1) * 3];
  memcpy(tmp, H, sizeof(double) * 3 * (n + 1));
  for (int c = 0; c < 3; c++) { L[c] = tmp[c]; R[3 * n + c] = tmp[3 * n + c]; }
  for (int r = 1; r <= n; r++) {
    for (int j = 0; j <= n - r; j++)
      for (int c = 0; c < 3; c++)
        tmp[3 * j + c] = 0.5 * (tmp[3 * j + c] + tmp[3 * (j + 1) + c]);
    for (int c = 0; c < 3; c++) {
      L[3 * r + c] = tmp[c];
      R[3 * (n - r) + c] = tmp[3 * (n - r) + c];
    }
  }
}

/* gamma(t) by homogeneous de Casteljau (any t in [0,1]); t==0 / t==1 return
 * the stored end control points exactly.  PINNED: S:54 worked value. */
void orc_eval(int n, const double *P, const double *w, double t, double *out) {
  if (t == 0.0) { out[0] = P[0]; out[1] = P[1]; return; }
  if (t == 1.0) { out[0] = P[2 * n]; out[1] = P[2 * n + 1]; return; }
  double H[(ORC_MAXDEG + 1) * 3];
  to_hom(n, P, w, H);
  for (int r = 1; r <= n; r++)
    for (int j = 0; j <= n - r; j++)
      for (int c = 0; c < 3; c++)
        H[3 * j + c] = (1.0 - t) * H[3 * j + c] + t * H[3 * (j + 1) + c];
  out[0] = H[0] / H[2];
  out[1] = H[1] / H[2];
}

/* gamma'(t) by the quotient rule on homogeneous de Casteljau values of the
 * curve and of its hodograph.  Used only to sample |gamma'| densely for the
 * derivative-bound soundness test (Lemma 1).  PINNED by comparison
 * with central finite differences in tests. */
void orc_deriv(int n, const double *P, const double *w, double t, double *out) {
  double H[(ORC_MAXDEG + 1) * 3], D[(ORC_MAXDEG + 1) * 3];
  to_hom(n, P, w, H);
  for (int j = 0; j < n; j++)
    for (int c = 0; c < 3; c++) D[3 * j + c] = n * (H[3 * (j + 1) + c] - H[3 * j + c]);
  for (int r = 1; r <= n; r++)
    for (int j = 0; j <= n - r; j++)
      for (int c = 0; c < 3; c++)
        H[3 * j + c] = (1.0 - t) * H[3 * j + c] + t * H[3 * (j + 1) + c];
  for (int r = 1; r <= n - 1; r++)
    for (int j = 0; j <= n - 1 - r; j++)
      for (int c = 0; c < 3; c++)
        D[3 * j + c] = (1.0 - t) * D[3 * j + c] + t * D[3 * (j + 1) + c];
  double X = H[0], Y = H[1], W = H[2];
  double dX = D[0], dY = D[1], dW = D[2];
  out[0] = (dX * W - X * dW) / (W * W);
  out[1] = (dY * W - Y * dW) / (W * W);
}

/* Adaptive subdivision of one piece.  ax..by are the piece's end points
 * (exact stored end points at the root, shared computed split points below,
 * so consecutive pieces telescope).  eta inflates boxes for the rounding of
 * the projected control points. */
static void seg_rec(int n, const double *H, double ax, double ay, double bx, double by,
                    double px, double py, double delta, double eta, int depth, acc_t *A) {
  double xmin = fmin(ax, bx), xmax = fmax(ax, bx), ymin = fmin(ay, by), ymax = fmax(ay, by);
  for (int j = 1; j < n; j++) {
    double x = H[3 * j] / H[3 * j + 2], y = H[3 * j + 1] / H[3 * j + 2];
    xmin = fmin(xmin, x); xmax = fmax(xmax, x);
    ymin = fmin(ymin, y); ymax = fmax(ymax, y);
  }
  xmin -= eta; ymin -= eta; xmax += eta; ymax += eta;
  double dx = fmax(fmax(xmin - px, px - xmax), 0.0);
  double dy = fmax(fmax(ymin - py, py - ymax), 0.0);
  double dist = hypot(dx, dy);
  if (dist > delta) {                         /* certified far: chord exact */
    nadd(A, orc_chord(px, py, ax, ay, bx, by));
    if (dist < A->dist_lb) A->dist_lb = dist;
    A->pieces++;
    return;
  }
  double diam = fmax(xmax - xmin, ymax - ymin);
  if (diam < 0.1 * delta || depth >= ORC_MAXDEPTH) {  /* near-curve: not comparable */
    A->near = 1;
    nadd(A, orc_chord(px, py, ax, ay, bx, by));
    if (dist < A->dist_lb) A->dist_lb = dist;
    A->pieces++;
    return;
  }
  double L[(ORC_MAXDEG + 1) * 3], R[(ORC_MAXDEG + 1) * 3];
  hsplit(n, H, L, R);
  double mx = L[3 * n] / L[3 * n + 2], my = L[3 * n + 1] / L[3 * n + 2];
  seg_rec(n, L, ax, ay, mx, my, px, py, delta, eta, depth + 1, A);
  seg_rec(n, R, mx, my, bx, by, px, py, delta, eta, depth + 1, A);
}

static double seg_eta(int n, const double *P) {
  double s = 1.0;
  for (int j = 0; j <= n; j++) s = fmax(s, fmax(fabs(P[2 * j]), fabs(P[2 * j + 1])));
  return 64.0 * 2.220446049250313e-16 * s;
}

/* Winding number of ONE (rational) Bezier segment about p by adaptive
 * de Casteljau + box-certified chords.  out[0]=omega, out[1]=near flag,
 * out[2]=dist_lb, out[3]=pieces. */
void orc_segment_winding(int n, const double *P, const double *w, double px, double py,
                         double delta, double *out) {
  double H[(ORC_MAXDEG + 1) * 3];
  to_hom(n, P, w, H);
  acc_t A;
  acc_init(&A);
  seg_rec(n, H, P[0], P[1], P[2 * n], P[2 * n + 1], px, py, delta, seg_eta(n, P), 0, &A);
  out[0] = acc_val(&A); out[1] = A.near; out[2] = A.dist_lb; out[3] = (double)A.pieces;
}

/* ------------------------------------------------------------------------ */
/* Face model: lifted loops                                                  */
/* ------------------------------------------------------------------------ */
typedef struct {
  int n_faces, n_loops, n_segs;
  const int *deg, *loop_off, *face_off;
  const uint8_t *per;
  const double *dom;
  /* lifted data (owned) */
  int64_t *ctrl_off;     /* [n_segs] offset (in points) into lifted ctrl */
  double *P;             /* lifted control points */
  double *H;             /* homogeneous, 3 per point */
  double *eta;           /* per segment */
  int *cls;              /* [n_loops*2] homology class (p,q) */
  double *bbox;          /* [n_loops*4] xmin ymin xmax ymax of lifted ctrl pts */
  int *pair_beta;        /* [n_loops] for alpha loops: paired beta loop, -1 none */
  int *pair_shift;       /* [n_loops*2] lattice shift (i,j) of the paired beta */
  int *face_err;         /* [n_faces] */
  int N5;                /* Eq. 5 truncation */
} model_t;

static inline double lat(double x, int k, double T) { return x + (double)k * T; }

/* Own lifting (R17/R18): segment i is translated by the lattice vector
 * k_i*T nearest to continuing from the lifted end of segment i-1; class =
 * round((end_last - start_0)/T) on periodic axes, 0 otherwise.  PINNED by the
 * SPEC homology examples S:281-283 and by the generators' known storage
 * shifts (tests/test_oracle_periodic.py). */
static void lift_all(model_t *M, const double *ctrl, const double *w, int *out_shift) {
  for (int l = 0; l < M->n_loops; l++) {
    int f = -1;
    /* find face of loop l */
    { int lo = 0, hi = M->n_faces - 1;
      while (lo < hi) { int mid = (lo + hi + 1) / 2; if (M->face_off[mid] <= l) lo = mid; else hi = mid - 1; }
      f = lo; }
    const double *D = M->dom + 4 * f;
    int pu = M->per[f] & 1, pv = (M->per[f] >> 1) & 1;
    int ku = 0, kv = 0;
    double endx = 0, endy = 0, sx = 0, sy = 0;
    double xmin = INFINITY, ymin = INFINITY, xmax = -INFINITY, ymax = -INFINITY;
    for (int s = M->loop_off[l]; s < M->loop_off[l + 1]; s++) {
      int n = M->deg[s];
      int64_t o = M->ctrl_off[s];
      const double *Ps = ctrl + 2 * o;
      if (s > M->loop_off[l]) {
        if (pu) ku = (int)round((endx - Ps[0]) / D[1]);
        if (pv) kv = (int)round((endy - Ps[1]) / D[3]);
      } else { ku = 0; kv = 0; }
      if (out_shift) { out_shift[2 * s] = ku; out_shift[2 * s + 1] = kv; }
      for (int j = 0; j <= n; j++) {
        double x = pu ? lat(Ps[2 * j], ku, D[1]) : Ps[2 * j];
        double y = pv ? lat(Ps[2 * j + 1], kv, D[3]) : Ps[2 * j + 1];
        M->P[2 * (o + j)] = x; M->P[2 * (o + j) + 1] = y;
        double wj = w ? w[o + j] : 1.0;
        M->H[3 * (o + j)] = wj * x; M->H[3 * (o + j) + 1] = wj * y; M->H[3 * (o + j) + 2] = wj;
        xmin = fmin(xmin, x); xmax = fmax(xmax, x); ymin = fmin(ymin, y); ymax = fmax(ymax, y);
      }
      if (s == M->loop_off[l]) { sx = M->P[2 * o]; sy = M->P[2 * o + 1]; }
      endx = M->P[2 * (o + n)]; endy = M->P[2 * (o + n) + 1];
      M->eta[s] = seg_eta(n, M->P + 2 * o);
    }
    M->cls[2 * l] = pu ? (int)round((endx - sx) / D[1]) : 0;
    M->cls[2 * l + 1] = pv ? (int)round((endy - sy) / D[3]) : 0;
    M->bbox[4 * l] = xmin; M->bbox[4 * l + 1] = ymin; M->bbox[4 * l + 2] = xmax; M->bbox[4 * l + 3] = ymax;
  }
}

/* omega(p, loop + (tx,ty)) via the translation identity omega(p, g+v) =
 * omega(p-v, g) (App. C.1). */
static void loop_wn(const model_t *M, int l, double px, double py, double delta, acc_t *A) {
  for (int s = M->loop_off[l]; s < M->loop_off[l + 1]; s++) {
    int n = M->deg[s];
    int64_t o = M->ctrl_off[s];
    const double *P = M->P + 2 * o;
    seg_rec(n, M->H + 3 * o, P[0], P[1], P[2 * n], P[2 * n + 1], px, py, delta, M->eta[s], 0, A);
  }
}

/* omega(p, L): +1/2 if p is left of the line through b0 with direction v
 * (cross(v, p-b0) >= 0, on L counts as left: R11), else -1/2. */
static double line_wn(double px, double py, double bx, double by, double vx, double vy) {
  double cr = vx * (py - by) - vy * (px - bx);
  return cr >= 0.0 ? 0.5 : -0.5;
}

/* Eq. 5 literally for the periodically extended curve of loop l
 * translated by (tx,ty), extension vector v = (vx,vy):
 *   sum_{k=kc-N..kc+N} omega(p, g_k) + omega(p,L) - omega(p, beta_{kc-N}, beta_{kc+N+1}),
 * g_k = g + k v, beta_k = g(0) + k v.  Translation applied to p (App. C.1).
 * The truncation window is centred on p's position along v (kc), so that the
 * copies which can wind around p are inside it whatever lattice representative
 * (tx,ty) of the extended curve is passed (Eq. 5 holds for any window that
 * contains them; the omitted copy-minus-chord loops do not enclose p). */
static void ext_wn(const model_t *M, int l, double tx, double ty, double vx, double vy,
                   double px, double py, double delta, acc_t *A) {
  int N = M->N5;
  int64_t o = M->ctrl_off[M->loop_off[l]];
  double b0x = M->P[2 * o] + tx, b0y = M->P[2 * o + 1] + ty;
  int kc = (int)round(((px - b0x) * vx + (py - b0y) * vy) / (vx * vx + vy * vy));
  for (int k = kc - N; k <= kc + N; k++)
    loop_wn(M, l, px - tx - k * vx, py - ty - k * vy, delta, A);
  nadd(A, line_wn(px, py, b0x, b0y, vx, vy));
  nadd(A, -orc_chord(px, py, b0x + (kc - N) * vx, b0y + (kc - N) * vy, b0x + (kc + N + 1) * vx,
                     b0y + (kc + N + 1) * vy));
}

static int gcd_i(int a, int b) { a = abs(a); b = abs(b); while (b) { int t = a % b; a = b; b = t; } return a; }

/* ToLeft (Alg. 7): is extended curve c1 (loop l1 shifted by
 * (t1x,t1y)) on the left of extended curve c2 (loop l2 shifted by
 * (t2x,t2y))?  Probe = c1's start point (a point of c1; the paper uses
 * gamma1(0.5), any point of a disjoint curve gives the same answer). */
static int to_left(const model_t *M, int l1, double t1x, double t1y, int l2, double t2x, double t2y,
                   double vx2, double vy2) {
  int64_t o = M->ctrl_off[M->loop_off[l1]];
  double qx = M->P[2 * o] + t1x, qy = M->P[2 * o + 1] + t1y;
  acc_t A;
  acc_init(&A);
  ext_wn(M, l2, t2x, t2y, vx2, vy2, qx, qy, 1e-12, &A);
  return acc_val(&A) > 0.0;
}

/* Band index of a bi-periodic face with non-contractible class (cp,cq)
 * (Prop. 2): nu(x) = cp*y/Tv - cq*x/Tu.  A lattice translate
 * (i Tu, j Tv) shifts nu by m = cp*j - cq*i, an integer; translates with the
 * same m differ by multiples of the extension vector v = (cp Tu, cq Tv) and
 * give the same extended curve, so the extended curves gamma_{r,s} of Eq. (8)
 * are indexed by m (gcd(cp,cq) = 1 makes every integer occur exactly once,
 * r in [0,|p|), s in Z).  rep_m returns one translate (i,j) with shift m. */
static double band_nu(int cp, int cq, const double *D, double x, double y) {
  return (double)cp * y / D[3] - (double)cq * x / D[1];
}
static void band_rep(int cp, int cq, int m, int *i, int *j) {
  /* extended Euclid: cp*y0 - cq*x0 = 1 */
  int r0 = cp, r1 = -cq, s0 = 1, s1 = 0, t0 = 0, t1 = 1;   /* s*cp + t*(-cq) = r */
  while (r1 != 0) {
    int qq = r0 / r1, tmp;
    tmp = r0 - qq * r1; r0 = r1; r1 = tmp;
    tmp = s0 - qq * s1; s0 = s1; s1 = tmp;
    tmp = t0 - qq * t1; t0 = t1; t1 = tmp;
  }
  if (r0 < 0) { s0 = -s0; t0 = -t0; }                     /* r0 = gcd = 1 */
  *j = m * s0; *i = m * t0;                                /* cp*j - cq*i = m */
}
/* nu-range of a loop's control-point box shifted by (i,j) tiles */
static void box_nu(const model_t *M, int l, int cp, int cq, const double *D, int i, int j,
                   double *lo, double *hi) {
  const double *bb = M->bbox + 4 * l;
  *lo = INFINITY; *hi = -INFINITY;
  for (int c = 0; c < 4; c++) {
    double x = bb[(c & 1) ? 2 : 0] + i * D[1], y = bb[(c & 2) ? 3 : 1] + j * D[3];
    double nu = band_nu(cp, cq, D, x, y);
    *lo = fmin(*lo, nu); *hi = fmax(*hi, nu);
  }
}

/* Validation (Props. 1, B.1, B.3 as input checks) and
 * pairing (Algs. 8-9, R16: search over the beta-translates modulo the
 * extension vector, i.e. over the band index m, in a window derived from the
 * loops' extents).  Error codes: 1 = |class|>1 on a uni-periodic axis (B.1),
 * 2 = unbalanced A/B (Prop. 1), 3 = mixed / non-coprime classes (B.3 / B.4),
 * 5 = pairing failure.  General classes (p,q), p,q != 0 (Prop. 2, Dataset B
 * P:804) are paired like the axis classes: the candidate translate of band m
 * is moved along v next to alpha (any representative gives the same extended
 * curve; a nearby one keeps the ToLeft probe inside Eq. 5's window). */
static void validate_and_pair(model_t *M) {
  for (int f = 0; f < M->n_faces; f++) {
    M->face_err[f] = 0;
    int pu = M->per[f] & 1, pv = (M->per[f] >> 1) & 1;
    const double *D = M->dom + 4 * f;
    int l0 = M->face_off[f], l1 = M->face_off[f + 1];
    int cp = 0, cq = 0, nA = 0, nB = 0;
    for (int l = l0; l < l1; l++) {
      M->pair_beta[l] = -1;
      int a = M->cls[2 * l], b = M->cls[2 * l + 1];
      if (a == 0 && b == 0) continue;
      if (pu && !pv && abs(a) > 1) M->face_err[f] = 1;
      if (pv && !pu && abs(b) > 1) M->face_err[f] = 1;
      if (gcd_i(a, b) != 1) M->face_err[f] = 3;
      if (cp == 0 && cq == 0) { cp = a; cq = b; }
      if (a == cp && b == cq) nA++;
      else if (a == -cp && b == -cq) nB++;
      else M->face_err[f] = 3;
    }
    if (M->face_err[f]) continue;
    if (nA != nB) { M->face_err[f] = 2; continue; }
    if (!(pu && pv) || nA == 0) continue;
    /* bi-periodic pairing.  Extension of A loops: v = (cp*Tu, cq*Tv). */
    double vAx = cp * D[1], vAy = cq * D[3];
    int general = (cp != 0 && cq != 0);
    int *used = (int *)calloc((size_t)(l1 - l0), sizeof(int));
    for (int la = l0; la < l1; la++) {
      if (!(M->cls[2 * la] == cp && M->cls[2 * la + 1] == cq)) continue;
      int best = -1, bi = 0, bj = 0;
      int64_t oa = M->ctrl_off[M->loop_off[la]];
      double sax = M->P[2 * oa], say = M->P[2 * oa + 1];
      double alo, ahi;
      box_nu(M, la, cp, cq, D, 0, 0, &alo, &ahi);
      for (int lb = l0; lb < l1; lb++) {
        if (used[lb - l0] || !(M->cls[2 * lb] == -cp && M->cls[2 * lb + 1] == -cq)) continue;
        /* window: translates whose transverse (nu) extent lies within 3 bands */
        double blo, bhi;
        box_nu(M, lb, cp, cq, D, 0, 0, &blo, &bhi);
        int J = 3 + (int)ceil((bhi - blo) + fabs(alo - blo));
        int64_t ob = M->ctrl_off[M->loop_off[lb]];
        for (int m = -J; m <= J; m++) {
          int i, j;
          band_rep(cp, cq, m, &i, &j);
          if (general) {   /* representative next to alpha along v */
            double dx = sax - (M->P[2 * ob] + i * D[1]), dy = say - (M->P[2 * ob + 1] + j * D[3]);
            int k = (int)round((dx * vAx + dy * vAy) / (vAx * vAx + vAy * vAy));
            i += k * cp; j += k * cq;
          }
          double tx = i * D[1], ty = j * D[3];
          if (!to_left(M, lb, tx, ty, la, 0.0, 0.0, vAx, vAy)) continue;
          if (best < 0 || to_left(M, lb, tx, ty, best, bi * D[1], bj * D[3], -vAx, -vAy)) {
            best = lb; bi = i; bj = j;
          }
        }
      }
      if (best < 0) { M->face_err[f] = 5; break; }
      used[best - l0] = 1;
      M->pair_beta[la] = best;
      M->pair_shift[2 * la] = bi;
      M->pair_shift[2 * la + 1] = bj;
    }
    free(used);
  }
}

/* winding of face f at p (p already reduced if requested) */
static void face_wn(const model_t *M, int f, double px, double py, double delta, acc_t *A) {
  const double *D = M->dom + 4 * f;
  int pu = M->per[f] & 1, pv = (M->per[f] >> 1) & 1;
  int l0 = M->face_off[f], l1 = M->face_off[f + 1];
  for (int l = l0; l < l1; l++) {
    int a = M->cls[2 * l], b = M->cls[2 * l + 1];
    const double *bb = M->bbox + 4 * l;
    if (!pu && !pv) { loop_wn(M, l, px, py, delta, A); continue; }
    if (a == 0 && b == 0) {
      /* contractible: all lattice translates within one period (plus a ring)
       * of p (Algs. 3/4) */
      int ilo = 0, ihi = 0, jlo = 0, jhi = 0;
      if (pu) { ilo = (int)floor((px - bb[2]) / D[1]) - 1; ihi = (int)ceil((px - bb[0]) / D[1]) + 1; }
      if (pv) { jlo = (int)floor((py - bb[3]) / D[3]) - 1; jhi = (int)ceil((py - bb[1]) / D[3]) + 1; }
      for (int i = ilo; i <= ihi; i++)
        for (int j = jlo; j <= jhi; j++)
          loop_wn(M, l, px - (pu ? i * D[1] : 0.0), py - (pv ? j * D[3] : 0.0), delta, A);
      continue;
    }
    double vx = a * D[1], vy = b * D[3];
    if (!(pu && pv)) { ext_wn(M, l, 0.0, 0.0, vx, vy, px, py, delta, A); continue; }
    /* bi-periodic: only alpha loops (class == face class A) drive Eq. 8
     * (P:583-590): sum over the bands m (the (r,s) of Eq. 8) of the extended
     * windings of alpha + rep(m) and of the proper beta-bar + rep(m), over
     * every band whose nu-extent lies within 3 bands of p. */
    if (M->pair_beta[l] < 0) continue;
    int lb = M->pair_beta[l];
    int si = M->pair_shift[2 * l], sj = M->pair_shift[2 * l + 1];
    double lo1, hi1, lo2, hi2;
    box_nu(M, l, a, b, D, 0, 0, &lo1, &hi1);
    box_nu(M, lb, a, b, D, si, sj, &lo2, &hi2);
    double lo = fmin(lo1, lo2), hi = fmax(hi1, hi2), c = band_nu(a, b, D, px, py);
    int mlo = (int)floor(c - hi) - 3, mhi = (int)ceil(c - lo) + 3;
    for (int m = mlo; m <= mhi; m++) {
      int i, j;
      band_rep(a, b, m, &i, &j);
      ext_wn(M, l, i * D[1], j * D[3], vx, vy, px, py, delta, A);
      ext_wn(M, lb, (si + i) * D[1], (sj + j) * D[3], -vx, -vy, px, py, delta, A);
    }
  }
}

static double round_half_away(double x) { return x >= 0 ? floor(x + 0.5) : -floor(-x + 0.5); }

/* Lifting only: per-segment integer shifts [n_segs][2] and per-loop classes
 * [n_loops][2]. */
int orc_lift(int n_faces, int n_loops, int n_segs, const double *ctrl_uv, const double *ctrl_w,
             const int *seg_degree, const int *loop_seg_off, const int *face_loop_off,
             const uint8_t *face_periodic, const double *face_domain, int *out_shift, int *out_class,
             double *out_bbox);

static int model_init(model_t *M, int n_faces, int n_loops, int n_segs, const double *ctrl_uv,
                      const double *ctrl_w, const int *seg_degree, const int *loop_seg_off,
                      const int *face_loop_off, const uint8_t *face_periodic,
                      const double *face_domain, int N5, int *out_shift) {
  memset(M, 0, sizeof(*M));
  M->n_faces = n_faces; M->n_loops = n_loops; M->n_segs = n_segs;
  M->deg = seg_degree; M->loop_off = loop_seg_off; M->face_off = face_loop_off;
  M->per = face_periodic; M->dom = face_domain; M->N5 = N5;
  M->ctrl_off = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n_segs + 1));
  int64_t o = 0;
  for (int s = 0; s < n_segs; s++) {
    if (seg_degree[s] < 1 || seg_degree[s] > ORC_MAXDEG) return -1;
    M->ctrl_off[s] = o; o += seg_degree[s] + 1;
  }
  M->ctrl_off[n_segs] = o;
  if (ctrl_w)
    for (int64_t i = 0; i < o; i++) if (!(ctrl_w[i] > 0.0)) return -2;
  M->P = (double *)malloc(sizeof(double) * 2 * (size_t)o);
  M->H = (double *)malloc(sizeof(double) * 3 * (size_t)o);
  M->eta = (double *)malloc(sizeof(double) * (size_t)n_segs);
  M->cls = (int *)malloc(sizeof(int) * 2 * (size_t)n_loops);
  M->bbox = (double *)malloc(sizeof(double) * 4 * (size_t)n_loops);
  M->pair_beta = (int *)malloc(sizeof(int) * (size_t)n_loops);
  M->pair_shift = (int *)calloc(2 * (size_t)n_loops, sizeof(int));
  M->face_err = (int *)calloc((size_t)n_faces, sizeof(int));
  lift_all(M, ctrl_uv, ctrl_w, out_shift);
  for (int l = 0; l < n_loops; l++) M->pair_beta[l] = -1;
  validate_and_pair(M);
  return 0;
}

static void model_free(model_t *M) {
  free(M->ctrl_off); free(M->P); free(M->H); free(M->eta); free(M->cls); free(M->bbox);
  free(M->pair_beta); free(M->pair_shift); free(M->face_err);
}

int orc_lift(int n_faces, int n_loops, int n_segs, const double *ctrl_uv, const double *ctrl_w,
             const int *seg_degree, const int *loop_seg_off, const int *face_loop_off,
             const uint8_t *face_periodic, const double *face_domain, int *out_shift, int *out_class,
             double *out_bbox) {
  model_t M;
  int rc = model_init(&M, n_faces, n_loops, n_segs, ctrl_uv, ctrl_w, seg_degree, loop_seg_off,
                      face_loop_off, face_periodic, face_domain, 4, out_shift);
  if (rc == 0) {
    if (out_class) memcpy(out_class, M.cls, sizeof(int) * 2 * (size_t)n_loops);
    if (out_bbox) memcpy(out_bbox, M.bbox, sizeof(double) * 4 * (size_t)n_loops);
  }
  model_free(&M);
  return rc;
}

/* Pairing result for tests: out_pair[n_loops] = paired beta (or -1),
 * out_pshift[n_loops*2], out_face_err[n_faces]. */
int orc_pairs(int n_faces, int n_loops, int n_segs, const double *ctrl_uv, const double *ctrl_w,
              const int *seg_degree, const int *loop_seg_off, const int *face_loop_off,
              const uint8_t *face_periodic, const double *face_domain, int N5, int *out_pair,
              int *out_pshift, int *out_face_err) {
  model_t M;
  int rc = model_init(&M, n_faces, n_loops, n_segs, ctrl_uv, ctrl_w, seg_degree, loop_seg_off,
                      face_loop_off, face_periodic, face_domain, N5, NULL);
  if (rc == 0) {
    memcpy(out_pair, M.pair_beta, sizeof(int) * (size_t)n_loops);
    memcpy(out_pshift, M.pair_shift, sizeof(int) * 2 * (size_t)n_loops);
    memcpy(out_face_err, M.face_err, sizeof(int) * (size_t)n_faces);
  }
  model_free(&M);
  return rc;
}

/* Batched query.  reduce=1 reduces periodic coordinates into the base tile
 * (u in [u0,u0+T) kept bit-exact).  rule 0 = nonzero, 1 = positive.
 * out_flag: 0 outside, 1 inside, 3 invalid query or invalid face.
 * Returns 0, or <0 on invalid geometry (degree / weight). */
int orc_query(int n_faces, int n_loops, int n_segs, const double *ctrl_uv, const double *ctrl_w,
              const int *seg_degree, const int *loop_seg_off, const int *face_loop_off,
              const uint8_t *face_periodic, const double *face_domain, int64_t nq,
              const int *face_id, const double *uv, double delta, double tol, int N5, int rule,
              int reduce, int strict, int nthreads, double *out_w, uint8_t *out_flag,
              uint8_t *out_cmp, double *out_distlb, int64_t *out_pieces, int *out_face_err) {
  model_t M;
  int rc = model_init(&M, n_faces, n_loops, n_segs, ctrl_uv, ctrl_w, seg_degree, loop_seg_off,
                      face_loop_off, face_periodic, face_domain, N5, NULL);
  if (rc != 0) { model_free(&M); return rc; }
  /* strict = 0: an unbalanced uni-periodic loop set (Prop. 1 violated, code 2)
   * is still evaluated -- used for the single-extended-curve worked values
   * which are primitives, not valid faces. */
  if (!strict)
    for (int f = 0; f < n_faces; f++)
      if (M.face_err[f] == 2 && !((face_periodic[f] & 3) == 3)) M.face_err[f] = 0;
  if (out_face_err) memcpy(out_face_err, M.face_err, sizeof(int) * (size_t)n_faces);
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 16)
#endif
  for (int64_t q = 0; q < nq; q++) {
    int f = face_id[q];
    double px = uv[2 * q], py = uv[2 * q + 1];
    if (f < 0 || f >= n_faces || !isfinite(px) || !isfinite(py) || M.face_err[f]) {
      out_w[q] = NAN; out_flag[q] = 3; out_cmp[q] = 0;
      if (out_distlb) out_distlb[q] = 0.0;
      if (out_pieces) out_pieces[q] = 0;
      continue;
    }
    const double *D = face_domain + 4 * f;
    if (reduce) {
      if ((face_periodic[f] & 1) && !(px >= D[0] && px < D[0] + D[1])) {
        px = D[0] + ((px - D[0]) - D[1] * floor((px - D[0]) / D[1]));
        if (px >= D[0] + D[1]) px = D[0];
      }
      if ((face_periodic[f] & 2) && !(py >= D[2] && py < D[2] + D[3])) {
        py = D[2] + ((py - D[2]) - D[3] * floor((py - D[2]) / D[3]));
        if (py >= D[2] + D[3]) py = D[2];
      }
    }
    acc_t A;
    acc_init(&A);
    face_wn(&M, f, px, py, delta, &A);
    double wv = acc_val(&A);
    double r = round_half_away(wv);
    out_w[q] = wv;
    out_flag[q] = (rule == 0) ? (fabs(r) >= 1.0) : (r >= 1.0);
    double fr = fabs(wv - floor(wv) - 0.5);   /* distance to nearest half-integer */
    out_cmp[q] = (!A.near && A.dist_lb > delta && fr > tol) ? 1 : 0;
    if (out_distlb) out_distlb[q] = A.dist_lb;
    if (out_pieces) out_pieces[q] = A.pieces;
  }
  model_free(&M);
  return 0;
}

/* ---------------------------------------------------------------------------
 * NURBS ingest ("B-spline or NURBS curves can always be subdivided
 * into (rational) Bezier segments"; SPEC decompose_bspline).  Plain repeated
 * single knot insertion (Boehm's rule in homogeneous coordinates (w x, w y,
 * w)): every distinct interior knot value of multiplicity s is inserted p - s
 * times; afterwards every interior knot has multiplicity p and the control
 * polygon splits into Bezier segments j = points [j p, j p + p].
 *   Single insertion of u with K[l] <= u < K[l+1] (NURBS Book eq. 5.15):
 *     Q_i = P_i                                  i <= l - p
 *     Q_i = a_i P_i + (1 - a_i) P_{i-1},          l-p+1 <= i <= l,
 *           a_i = (u - K[i]) / (K[i+p] - K[i])
 *     Q_i = P_{i-1}                              i >= l + 1
 * PINNED (tests/test_oracle_nurbs.py) by an independent Cox-de Boor evaluation
 * of the spline at random parameters, SPEC's single-span / two-span examples
 * and the exact 9-point NURBS circle.
 * Input: degree p (1..5), n_ctrl points P[n_ctrl][2], weights w (NULL = 1),
 * knots U[n_ctrl + p + 1] (clamped, non-decreasing, interior multiplicity <= p).
 * Output: up to cap segments of p+1 points (outP [seg][p+1][2], outw
 * [seg][p+1]; the curve's two end points are copied from P exactly); returns the number of segments, -1 invalid knots, -2 cap too
 * small, -3 bad degree / weight. */
int orc_nurbs_decompose(int p, int n_ctrl, const double *P, const double *w, const double *U, int cap,
                        double *outP, double *outw) {
  if (p < 1 || p > ORC_MAXDEG || n_ctrl < p + 1) return -3;
  int nk = n_ctrl + p + 1;
  for (int i = 0; i + 1 < nk; i++) if (!(U[i] <= U[i + 1])) return -1;
  for (int i = 1; i <= p; i++) if (U[i] != U[0] || U[nk - 1 - i] != U[nk - 1]) return -1;
  if (!(U[p] < U[nk - 1 - p])) return -1;
  /* clamped means EXACTLY p+1 equal end knots (a (p+2)-fold end knot is not a
   * clamped knot vector of this degree: the Bezier form's end points would no
   * longer be P_0 / P_n) */
  if (U[p + 1] == U[p] || U[nk - 2 - p] == U[nk - 1 - p]) return -1;
  for (int i = p + 1; i < nk - 1 - p; i++) {        /* interior multiplicity <= p */
    int s = 1;
    while (i + s < nk - 1 - p && U[i + s] == U[i]) s++;
    if (s > p) return -1;
    i += s - 1;
  }
  if (w) for (int i = 0; i < n_ctrl; i++) if (!(w[i] > 0.0)) return -3;
  int maxn = n_ctrl + p * nk;                       /* room for all insertions */
  double *H = (double *)malloc(sizeof(double) * 3 * (size_t)maxn);
  double *H2 = (double *)malloc(sizeof(double) * 3 * (size_t)maxn);
  double *K = (double *)malloc(sizeof(double) * (size_t)(nk + p * nk));
  for (int i = 0; i < n_ctrl; i++) {
    double wi = w ? w[i] : 1.0;
    H[3 * i] = wi * P[2 * i]; H[3 * i + 1] = wi * P[2 * i + 1]; H[3 * i + 2] = wi;
  }
  memcpy(K, U, sizeof(double) * (size_t)nk);
  int n = n_ctrl, m = nk;
  double u_end = U[nk - 1 - p];
  int i = p + 1;
  while (K[i] < u_end) {
    double u = K[i];
    int s = 0;
    while (K[i + s] == u) s++;
    for (int r = 0; r < p - s; r++) {
      int l = i + s - 1 + r;                         /* last index with K[l] <= u */
      for (int j = 0; j <= n; j++) {
        if (j <= l - p) { memcpy(H2 + 3 * j, H + 3 * j, 3 * sizeof(double)); }
        else if (j >= l + 1) { memcpy(H2 + 3 * j, H + 3 * (j - 1), 3 * sizeof(double)); }
        else {
          double a = (u - K[j]) / (K[j + p] - K[j]);
          for (int c = 0; c < 3; c++) H2[3 * j + c] = a * H[3 * j + c] + (1.0 - a) * H[3 * (j - 1) + c];
        }
      }
      double *t = H; H = H2; H2 = t;
      n++;
      memmove(K + l + 2, K + l + 1, sizeof(double) * (size_t)(m - l - 1));
      K[l + 1] = u;
      m++;
    }
    i += p;                                          /* now multiplicity p */
  }
  int nseg = (n - 1) / p;
  int rc = nseg;
  if (nseg > cap) rc = -2;
  else
    for (int sgi = 0; sgi < nseg; sgi++)
      for (int j = 0; j <= p; j++) {
        const double *h = H + 3 * (sgi * p + j);
        outw[sgi * (p + 1) + j] = h[2];
        outP[2 * (sgi * (p + 1) + j)] = h[0] / h[2];
        outP[2 * (sgi * (p + 1) + j) + 1] = h[1] / h[2];
      }
  if (rc > 0) {
    /* the curve's end points are P_0 and P_n exactly (clamped knots): keep
     * them bit-identical (junctions with the neighbouring curves of a loop) */
    outP[0] = P[0]; outP[1] = P[1]; outw[0] = w ? w[0] : 1.0;
    int e = (nseg - 1) * (p + 1) + p;
    outP[2 * e] = P[2 * (n_ctrl - 1)]; outP[2 * e + 1] = P[2 * (n_ctrl - 1) + 1];
    outw[e] = w ? w[n_ctrl - 1] : 1.0;
  }
  free(H); free(H2); free(K);
  return rc;
}
