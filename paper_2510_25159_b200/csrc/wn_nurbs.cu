// wn_nurbs.cu -- NURBS p-curve ingest.
//
// The paper represents p-curves as (rational) Bezier or NURBS curves and notes
// that "B-spline or NURBS curves can always be subdivided into (rational)
// Bezier segments"; its future-work paragraph leaves a
// linear NURBS evaluation open.  This file performs that subdivision on the
// device so NURBS trimming loops feed the Bezier build (wn_build_faces) with no
// host round trip: one thread per curve runs the classic curve decomposition
// (knot insertion of every interior knot up to multiplicity p, sweeping the
// knot vector once, homogeneous coordinates (w x, w y, w)), writing each
// Bezier segment as soon as it is complete.
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "wn_common.cuh"

namespace wn {

namespace {

// Validation + segment count of one curve: clamped (exactly p+1 equal end knots),
// non-decreasing, U[p] < U[m-p], interior multiplicity <= p, finite data,
// positive weights.  Segments = distinct interior knot values + 1.
__global__ void k_nurbs_count(int32_t n_curves, int32_t n_ctrl_total, int32_t n_knots_total,
                              const double *__restrict__ ctrl, const double *__restrict__ w,
                              const int32_t *__restrict__ deg, const int32_t *__restrict__ coff,
                              const double *__restrict__ knots, const int32_t *__restrict__ koff,
                              int32_t *__restrict__ nseg, int32_t *__restrict__ npts, int32_t *__restrict__ bad) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c > n_curves) return;
  if (c == n_curves) { nseg[c] = 0; npts[c] = 0; return; }
  nseg[c] = 0;
  npts[c] = 0;
  const int p = deg[c];
  const int c0 = coff[c], c1 = coff[c + 1], k0 = koff[c], k1 = koff[c + 1];
  const int nc = c1 - c0, nk = k1 - k0;
  bool ok = p >= 1 && p <= 5 && c0 >= 0 && c1 <= n_ctrl_total && k0 >= 0 && k1 <= n_knots_total &&
            nc >= p + 1 && nk == nc + p + 1;
  if (!ok) { atomicMin(bad, c); return; }
  const double *U = knots + k0;
  for (int i = 0; i < nk; ++i) ok &= isfinite(U[i]) && (i == 0 || U[i - 1] <= U[i]);
  for (int i = 1; i <= p && ok; ++i) ok &= U[i] == U[0] && U[nk - 1 - i] == U[nk - 1];
  ok &= U[p] < U[nk - 1 - p];
  // exactly p+1 equal end knots: a (p+2)-fold end knot would be counted as an
  // interior knot here while the fill sweep runs into the end knots
  ok &= U[p + 1] != U[p] && U[nk - 2 - p] != U[nk - 1 - p];
  int count = 1;
  for (int i = p + 1; i < nk - 1 - p && ok;) {
    int s = 1;
    while (i + s < nk - 1 - p && U[i + s] == U[i]) ++s;
    ok &= s <= p;
    ++count;
    i += s;
  }
  for (int i = c0; i < c1 && ok; ++i) {
    ok &= isfinite(ctrl[2 * i]) && isfinite(ctrl[2 * i + 1]);
    if (w) ok &= w[i] > 0.0 && isfinite(w[i]);
  }
  if (!ok) { atomicMin(bad, c); return; }
  nseg[c] = count;
  npts[c] = count * (p + 1);
}

// Decomposition of one curve (one thread): sweep the distinct interior knots
// in order; at each, insert it until it has multiplicity p (the new points
// of the current segment are blended in place right to left, and the first
// points of the next segment are saved as they appear), emit the completed
// segment, then start the next one from the saved points and the untouched
// original control points.
__global__ void k_nurbs_fill(int32_t n_curves, const double *__restrict__ ctrl, const double *__restrict__ w,
                             const int32_t *__restrict__ deg, const int32_t *__restrict__ coff,
                             const double *__restrict__ knots, const int32_t *__restrict__ koff,
                             const int32_t *__restrict__ seg_off, const int32_t *__restrict__ pt_off,
                             double *__restrict__ bez, double *__restrict__ bw, int32_t *__restrict__ bdeg) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n_curves) return;
  const int p = deg[c];
  const int c0 = coff[c], nc = coff[c + 1] - c0;
  const double *U = knots + koff[c];
  const int m = nc + p;                       // last knot index
  const int nseg = seg_off[c + 1] - seg_off[c];
  if (nseg <= 0) return;
  double Q[6][3], N[6][3], alpha[6];
  auto load = [&](int i, double *o) {
    const double wi = w ? w[c0 + i] : 1.0;
    o[0] = wi * ctrl[2 * (c0 + i)];
    o[1] = wi * ctrl[2 * (c0 + i) + 1];
    o[2] = wi;
  };
  for (int i = 0; i <= p; ++i) load(i, Q[i]);
  int a = p, b = p + 1, sg = 0;
  int out = pt_off[c];
  while (b < m) {
    const int i0 = b;
    while (b < m && U[b + 1] == U[b]) ++b;
    const int mult = b - i0 + 1;
    int r = 0;
    if (mult < p) {
      const double numer = U[b] - U[a];
      for (int j = p; j > mult; --j) alpha[j - mult - 1] = numer / (U[a + j] - U[a]);
      r = p - mult;
      for (int j = 1; j <= r; ++j) {
        const int save = r - j, s = mult + j;
        for (int k = p; k >= s; --k) {
          const double al = alpha[k - s];
          for (int d = 0; d < 3; ++d) Q[k][d] = al * Q[k][d] + (1.0 - al) * Q[k - 1][d];
        }
        if (b < m)
          for (int d = 0; d < 3; ++d) N[save][d] = Q[p][d];
      }
    }
    // emit segment sg (the curve's first point is the input point, bit-exact)
    for (int j = 0; j <= p; ++j, ++out) {
      if (sg == 0 && j == 0) {
        bez[2 * out] = ctrl[2 * c0];
        bez[2 * out + 1] = ctrl[2 * c0 + 1];
        bw[out] = w ? w[c0] : 1.0;
      } else {
        bez[2 * out] = Q[j][0] / Q[j][2];
        bez[2 * out + 1] = Q[j][1] / Q[j][2];
        bw[out] = Q[j][2];
      }
    }
    bdeg[seg_off[c] + sg] = p;
    ++sg;
    if (b < m) {
      for (int i = p - mult; i <= p; ++i) load(b - p + i, N[i]);
      for (int i = 0; i <= p; ++i)
        for (int d = 0; d < 3; ++d) Q[i][d] = N[i][d];
      a = b;
      ++b;
    }
  }
  // the curve's last point is the input point, bit-exact (clamped knots)
  const int e = out - 1;
  bez[2 * e] = ctrl[2 * (c0 + nc - 1)];
  bez[2 * e + 1] = ctrl[2 * (c0 + nc - 1) + 1];
  bw[e] = w ? w[c0 + nc - 1] : 1.0;
}

__global__ void k_loop_segs(int32_t n_loops, const int32_t *__restrict__ loop_curve_off,
                            const int32_t *__restrict__ seg_off, int32_t *__restrict__ loop_seg_off) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l <= n_loops) loop_seg_off[l] = seg_off[loop_curve_off[l]];
}

struct Decomp {
  int32_t *seg_off = nullptr, *pt_off = nullptr, *bdeg = nullptr;
  double *bez = nullptr, *bw = nullptr;
  int32_t n_segs = 0, n_pts = 0;
};

// count, scan, (host reads the totals), fill into library-owned buffers
wn_status_t decompose(int32_t n_curves, int32_t n_ctrl, int32_t n_knots, const double *ctrl, const double *w,
                      const int32_t *deg, const int32_t *coff, const double *knots, const int32_t *koff,
                      cudaStream_t st, Decomp &D, int &launches) {
  int32_t *nseg = nullptr, *npts = nullptr, *bad = nullptr;
  WN_CUDA(cache_alloc((void **)&nseg, sizeof(int32_t) * (n_curves + 1), st));
  WN_CUDA(cache_alloc((void **)&npts, sizeof(int32_t) * (n_curves + 1), st));
  WN_CUDA(cache_alloc((void **)&D.seg_off, sizeof(int32_t) * (n_curves + 1), st));
  WN_CUDA(cache_alloc((void **)&D.pt_off, sizeof(int32_t) * (n_curves + 1), st));
  WN_CUDA(cache_alloc((void **)&bad, sizeof(int32_t) * 4, st));
  const int32_t init = INT32_MAX;
  WN_CUDA(cudaMemcpyAsync(bad, &init, sizeof(int32_t), cudaMemcpyHostToDevice, st));
  k_nurbs_count<<<(n_curves + 128) / 128, 128, 0, st>>>(n_curves, n_ctrl, n_knots, ctrl, w, deg, coff, knots, koff,
                                                        nseg, npts, bad);
  ++launches;
  size_t tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, nseg, D.seg_off, n_curves + 1, st);
  void *tb = nullptr;
  WN_CUDA(cache_alloc(&tb, tmp, st));
  cub::DeviceScan::ExclusiveSum(tb, tmp, nseg, D.seg_off, n_curves + 1, st);
  cub::DeviceScan::ExclusiveSum(tb, tmp, npts, D.pt_off, n_curves + 1, st);
  launches += 4;
  int32_t hv[3];
  WN_CUDA(cudaMemcpyAsync(&hv[0], D.seg_off + n_curves, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  WN_CUDA(cudaMemcpyAsync(&hv[1], D.pt_off + n_curves, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  WN_CUDA(cudaMemcpyAsync(&hv[2], bad, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  WN_CUDA(cudaStreamSynchronize(st));
  cache_free(tb, st);
  cache_free(nseg, st);
  cache_free(npts, st);
  cache_free(bad, st);
  if (hv[2] != INT32_MAX) {
    set_error("NURBS curve %d invalid (degree 1..5, clamped non-decreasing knots, n_knots = n_ctrl + p + 1, "
              "interior multiplicity <= p, finite data, weights > 0)", hv[2]);
    return WN_ERR_GEOM;
  }
  D.n_segs = hv[0];
  D.n_pts = hv[1];
  WN_CUDA(cache_alloc((void **)&D.bez, sizeof(double) * 2 * std::max(D.n_pts, 1), st));
  WN_CUDA(cache_alloc((void **)&D.bw, sizeof(double) * std::max(D.n_pts, 1), st));
  WN_CUDA(cache_alloc((void **)&D.bdeg, sizeof(int32_t) * std::max(D.n_segs, 1), st));
  if (n_curves) {
    k_nurbs_fill<<<(n_curves + 127) / 128, 128, 0, st>>>(n_curves, ctrl, w, deg, coff, knots, koff, D.seg_off,
                                                         D.pt_off, D.bez, D.bw, D.bdeg);
    ++launches;
  }
  WN_CUDA(cudaGetLastError());
  return WN_OK;
}

void release(Decomp &D, cudaStream_t st) {
  for (void *p : {(void *)D.seg_off, (void *)D.pt_off, (void *)D.bez, (void *)D.bw, (void *)D.bdeg})
    if (p) cache_free(p, st);
  D = Decomp();
}

bool host_csr(const int32_t *d, int32_t n, int32_t last, cudaStream_t st, const char *what) {
  std::vector<int32_t> h(n + 1);
  if (cudaMemcpyAsync(h.data(), d, sizeof(int32_t) * (n + 1), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess) {
    set_error("%s: copy failed", what);
    return false;
  }
  if (h[0] != 0 || h[n] != last) { set_error("%s: CSR must start at 0 and end at %d", what, last); return false; }
  for (int i = 0; i < n; ++i)
    if (h[i] > h[i + 1]) { set_error("%s: CSR not non-decreasing at %d", what, i); return false; }
  return true;
}

}  // namespace
}  // namespace wn

using namespace wn;

extern "C" wn_status_t wn_nurbs_to_bezier(int32_t n_curves, int32_t n_ctrl, int32_t n_knots, const double *ctrl_uv,
                                          const double *ctrl_w, const int32_t *curve_degree,
                                          const int32_t *curve_ctrl_off, const double *knots,
                                          const int32_t *curve_knot_off, int32_t seg_cap, int32_t pt_cap,
                                          int32_t *curve_seg_off, double *bez_uv, double *bez_w,
                                          int32_t *bez_degree, int32_t *n_segs_out, int32_t *n_pts_out,
                                          void *stream) {
  set_error("");
  if (n_curves < 0 || n_ctrl < 0 || n_knots < 0 || seg_cap < 0 || pt_cap < 0) {
    set_error("wn_nurbs_to_bezier: negative size");
    return WN_ERR_ARG;
  }
  if (n_curves > 0 && (!ctrl_uv || !curve_degree || !curve_ctrl_off || !knots || !curve_knot_off ||
                       !curve_seg_off || !bez_uv || !bez_w || !bez_degree)) {
    set_error("wn_nurbs_to_bezier: NULL array");
    return WN_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  int dev = 0;
  WN_CUDA(cudaGetDevice(&dev));
  ensure_pool(dev);
  if (n_curves == 0) {
    if (n_segs_out) *n_segs_out = 0;
    if (n_pts_out) *n_pts_out = 0;
    if (curve_seg_off) WN_CUDA(cudaMemsetAsync(curve_seg_off, 0, sizeof(int32_t), st));
    return WN_OK;
  }
  if (!host_csr(curve_ctrl_off, n_curves, n_ctrl, st, "curve_ctrl_off") ||
      !host_csr(curve_knot_off, n_curves, n_knots, st, "curve_knot_off"))
    return WN_ERR_ARG;
  Decomp D;
  int launches = 0;
  wn_status_t rc = decompose(n_curves, n_ctrl, n_knots, ctrl_uv, ctrl_w, curve_degree, curve_ctrl_off, knots,
                             curve_knot_off, st, D, launches);
  if (rc != WN_OK) { release(D, st); return rc; }
  if (n_segs_out) *n_segs_out = D.n_segs;
  if (n_pts_out) *n_pts_out = D.n_pts;
  if (D.n_segs > seg_cap || D.n_pts > pt_cap) {
    set_error("wn_nurbs_to_bezier: capacity too small (need %d segments, %d points)", D.n_segs, D.n_pts);
    release(D, st);
    return WN_ERR_ARG;
  }
  WN_CUDA(cudaMemcpyAsync(curve_seg_off, D.seg_off, sizeof(int32_t) * (n_curves + 1), cudaMemcpyDeviceToDevice, st));
  WN_CUDA(cudaMemcpyAsync(bez_uv, D.bez, sizeof(double) * 2 * D.n_pts, cudaMemcpyDeviceToDevice, st));
  WN_CUDA(cudaMemcpyAsync(bez_w, D.bw, sizeof(double) * D.n_pts, cudaMemcpyDeviceToDevice, st));
  WN_CUDA(cudaMemcpyAsync(bez_degree, D.bdeg, sizeof(int32_t) * D.n_segs, cudaMemcpyDeviceToDevice, st));
  release(D, st);
  return WN_OK;
}

extern "C" wn_status_t wn_build_faces_nurbs(int32_t n_faces, int32_t n_loops, int32_t n_curves, int32_t n_ctrl,
                                            int32_t n_knots, const double *ctrl_uv, const double *ctrl_w,
                                            const int32_t *curve_degree, const int32_t *curve_ctrl_off,
                                            const double *knots, const int32_t *curve_knot_off,
                                            const int32_t *loop_curve_off, const int32_t *face_loop_off,
                                            const uint8_t *face_periodic, const double *face_domain,
                                            const wn_options_t *opts, void *stream, wn_faces_t *out,
                                            int32_t *face_status) {
  set_error("");
  if (!out) { set_error("wn_build_faces_nurbs: out == NULL"); return WN_ERR_ARG; }
  if (n_faces < 0 || n_loops < 0 || n_curves < 0 || n_ctrl < 0 || n_knots < 0) {
    set_error("wn_build_faces_nurbs: negative count");
    return WN_ERR_ARG;
  }
  if (!loop_curve_off || (n_curves > 0 && (!ctrl_uv || !curve_degree || !curve_ctrl_off || !knots ||
                                          !curve_knot_off))) {
    set_error("wn_build_faces_nurbs: NULL array");
    return WN_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  int dev = 0;
  WN_CUDA(cudaGetDevice(&dev));
  ensure_pool(dev);
  if (!host_csr(loop_curve_off, n_loops, n_curves, st, "loop_curve_off")) return WN_ERR_ARG;
  if (n_curves > 0 && (!host_csr(curve_ctrl_off, n_curves, n_ctrl, st, "curve_ctrl_off") ||
                       !host_csr(curve_knot_off, n_curves, n_knots, st, "curve_knot_off")))
    return WN_ERR_ARG;
  Decomp D;
  int launches = 0;
  int32_t *lso = nullptr;
  WN_CUDA(cache_alloc((void **)&lso, sizeof(int32_t) * (n_loops + 1), st));
  if (n_curves > 0) {
    wn_status_t rc = decompose(n_curves, n_ctrl, n_knots, ctrl_uv, ctrl_w, curve_degree, curve_ctrl_off, knots,
                               curve_knot_off, st, D, launches);
    if (rc != WN_OK) { release(D, st); cache_free(lso, st); return rc; }
    k_loop_segs<<<(n_loops + 128) / 128, 128, 0, st>>>(n_loops, loop_curve_off, D.seg_off, lso);
    ++launches;
  } else {
    WN_CUDA(cudaMemsetAsync(lso, 0, sizeof(int32_t) * (n_loops + 1), st));
  }
  // the Bezier build reads the decomposition asynchronously on `st`; the
  // stream-ordered frees below keep the buffers alive until it has
  const wn_status_t rc = wn_build_faces(n_faces, n_loops, D.n_segs, D.bez, D.bw, D.bdeg, lso, face_loop_off,
                                        face_periodic, face_domain, opts, stream, out, face_status);
  release(D, st);
  cache_free(lso, st);
  return rc;
}
