
#include <cstdio>
#include <cstdint>
#include <cmath>
struct SegPrep { double B, S0; double Bq[8]; };
// Exact binomial coefficients C(n,k), n <= 10.
__constant__ double c_binom[11][11] = {
    {1}, {1, 1}, {1, 2, 1}, {1, 3, 3, 1}, {1, 4, 6, 4, 1}, {1, 5, 10, 10, 5, 1}, {1, 6, 15, 20, 15, 6, 1},
    {1, 7, 21, 35, 35, 21, 7, 1}, {1, 8, 28, 56, 70, 56, 28, 8, 1}, {1, 9, 36, 84, 126, 126, 84, 36, 9, 1},
    {1, 10, 45, 120, 210, 252, 210, 120, 45, 10, 1}};

// Bounds on flat homogeneous control points H[3i+0..2] = (w x, w y, w), i = 0..n.
// Written without local aggregates (nvcc 12.9 -O3 miscompiled an earlier
// array-accumulating version on sm_100a; scripts/dev/kp.cu reproduces it).
// Hodograph-numerator Bernstein bound: max_k |D_k| / min_k E_k with
//   D_k = sum_{i+j=k} C(n-1,i)C(n,j)/C(2n-1,k) w_j (w_{i+1}(P_{i+1}-P_j) - w_i(P_i-P_j)),
//   E_k = sum_{i+j=k} C(n,i)C(n,j)/C(2n,k) w_i w_j.
__device__ __noinline__ double hodo_bound(int n, const double *H) {
  double dmax = 0.0, emin = INFINITY;
  for (int k = 0; k <= 2 * n - 1; ++k) {
    double dx = 0.0, dy = 0.0;
    const int i0 = k - n > 0 ? k - n : 0, i1 = k < n - 1 ? k : n - 1;
    for (int i = i0; i <= i1; ++i) {
      const int j = k - i;
      const double wi = H[3 * i + 2], wi1 = H[3 * i + 5], wj = H[3 * j + 2];
      const double xi = H[3 * i] / wi, yi = H[3 * i + 1] / wi;
      const double xi1 = H[3 * i + 3] / wi1, yi1 = H[3 * i + 4] / wi1;
      const double xj = H[3 * j] / wj, yj = H[3 * j + 1] / wj;
      const double c = c_binom[n - 1][i] * c_binom[n][j] / c_binom[2 * n - 1][k] * wj;
      dx += c * (wi1 * (xi1 - xj) - wi * (xi - xj));
      dy += c * (wi1 * (yi1 - yj) - wi * (yi - yj));
    }
    dmax = fmax(dmax, hypot(dx, dy));
  }
  for (int k = 0; k <= 2 * n; ++k) {
    double e = 0.0;
    const int i0 = k - n > 0 ? k - n : 0, i1 = k < n ? k : n;
    for (int i = i0; i <= i1; ++i) {
      const int j = k - i;
      e += c_binom[n][i] * c_binom[n][j] / c_binom[2 * n][k] * H[3 * i + 2] * H[3 * j + 2];
    }
    emin = fmin(emin, e);
  }
  return n * dmax / emin;
}

__device__ __noinline__ double floater_bound(int n, const double *H) {
  double wmax = H[2], wmin = H[2], dmax = 0.0, diam = 0.0;
  for (int i = 1; i <= n; ++i) { wmax = fmax(wmax, H[3 * i + 2]); wmin = fmin(wmin, H[3 * i + 2]); }
  for (int i = 0; i <= n; ++i)
    for (int j = i + 1; j <= n; ++j) {
      const double l = hypot(H[3 * j] / H[3 * j + 2] - H[3 * i] / H[3 * i + 2],
                             H[3 * j + 1] / H[3 * j + 2] - H[3 * i + 1] / H[3 * i + 2]);
      diam = fmax(diam, l);
      if (j == i + 1) dmax = fmax(dmax, l);
    }
  if (wmax == wmin) return n * dmax;
  const double r = wmax / wmin;
  return fmin(n * r * diam, n * r * r * dmax);
}

// Homogeneous control points of the dyadic piece [q/8, (q+1)/8] of H (blossom-
// free: three de Casteljau halvings, choosing the half along the bits of q).
// A receives 3(n+1) values; works in place in A.
__device__ __noinline__ void dyadic_piece(int n, const double *H, int q, double *A) {
  for (int i = 0; i < 3 * (n + 1); ++i) A[i] = H[i];
  for (int lvl = 2; lvl >= 0; --lvl) {
    const bool right = (q >> lvl) & 1;
    // after r rounds of midpoint averaging, entry 0 is the left half's point r
    // and entry n-r the right half's point n-r; keep the requested half
    double L[18], R[18];
    for (int c = 0; c < 3; ++c) { L[c] = A[c]; R[3 * n + c] = A[3 * n + c]; }
    for (int r = 1; r <= n; ++r) {
      for (int j = 0; j <= n - r; ++j)
        for (int c = 0; c < 3; ++c) A[3 * j + c] = 0.5 * (A[3 * j + c] + A[3 * j + 3 + c]);
      for (int c = 0; c < 3; ++c) { L[3 * r + c] = A[c]; R[3 * (n - r) + c] = A[3 * (n - r) + c]; }
    }
    for (int i = 0; i < 3 * (n + 1); ++i) A[i] = right ? R[i] : L[i];
  }
}

__global__ void k_prep(int32_t n_segs, const int32_t *__restrict__ deg, const int32_t *__restrict__ coff,
                       const double *__restrict__ ctrl, const double *__restrict__ w,
                       SegPrep *__restrict__ prep, uint8_t *__restrict__ serr) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_segs) return;
  const int n = deg[s];
  const int o = coff[s];
  double H[18], A[18];
  bool err = false;
  double lpoly = 0.0;
  for (int j = 0; j <= n; ++j) {
    const double x = ctrl[2 * (o + j)], y = ctrl[2 * (o + j) + 1], wj = w ? w[o + j] : 1.0;
    err |= !isfinite(x) || !isfinite(y) || !isfinite(wj) || !(wj > 0.0);
    H[3 * j] = wj * x; H[3 * j + 1] = wj * y; H[3 * j + 2] = wj;
    if (j) lpoly += hypot(x - ctrl[2 * (o + j - 1)], y - ctrl[2 * (o + j - 1) + 1]);
  }
  SegPrep *out = prep + s;
  if (err) {
    out->B = out->S0 = 0.0;
    for (int q = 0; q < 8; ++q) out->Bq[q] = 0.0;
  } else {
    const double B = fmin(floater_bound(n, H), hodo_bound(n, H));
    out->B = B;
    out->S0 = fmin(B, lpoly);
    for (int q = 0; q < 8; ++q) {
      dyadic_piece(n, H, q, A);
      out->Bq[q] = fmin(B, 8.0 * fmin(floater_bound(n, A), hodo_bound(n, A)));
    }
  }
  serr[s] = err ? 1 : 0;
}

int main(){
  const int ns = 5; int deg[ns] = {4,4,4,4,4}; double c[] = {0.7323866072190339,0.8477911355302876,0.7100677728912016,0.8543896424738517,0.6878369347685743,0.8550034201444957,0.6658615084526277,0.8382463292359036,0.6435185658675137,0.8464844681696877,0.2933251059855837,0.8093108373802549,0.2775534139051157,0.7962029754130869,0.25750626333615234,0.7933120168032823,0.24035123525980592,0.783509861164145,0.22096826549858983,0.7790317345014102,0.6874827104335929,0.4149219588763748,0.6937863595604539,0.40764433681140566,0.7026026241583173,0.40271781056725314,0.7053719763394085,0.3921330884407656,0.7137767512680147,0.386821524512628,0.8809289707399454,0.5,0.8858032697434884,0.5190762258220413,0.8856269566751688,0.5378539775896324,0.8745847664981038,0.5559895928498738,0.876503158528467,0.574891134588816,0.876503158528467,0.574891134588816,0.8789548081210381,0.5971413024501259,0.8799707292715993,0.619657567257674,0.8903377603091911,0.6404407036322465,0.8927763514303753,0.6626932917418824}; double w[] = {1.1688048191228209,0.977589498595514,0.5735200843446382,1.084392926448233,1.0490585858932073,0.7888924630685301,1.3230370639864897,0.9339168861828788,0.6582207153000603,0.5047801559271756,1.6972324190576884,1.9963410972974525,0.5559245037203362,1.1347241127967551,1.5613119602130046,1.184645931322334,1.8466012206397633,1.7527748070384195,1.077642701721225,1.9605181545578345,0.794254867952408,0.7576655226227518,0.7718093393464802,1.4057082758936579,0.6689492826669774};
  int coff[ns+1]; coff[0]=0; for(int i=0;i<ns;i++) coff[i+1]=coff[i]+deg[i]+1;
  int *dd, *dco; double *dc, *dw; SegPrep* dp; uint8_t* de;
  cudaMalloc(&dd, sizeof(deg)); cudaMalloc(&dco, sizeof(coff)); cudaMalloc(&dc, sizeof(c)); cudaMalloc(&dw, sizeof(w)); cudaMalloc(&dp, ns*sizeof(SegPrep)); cudaMalloc(&de, ns);
  cudaMemcpy(dd, deg, sizeof(deg), cudaMemcpyHostToDevice); cudaMemcpy(dco, coff, sizeof(coff), cudaMemcpyHostToDevice);
  cudaMemcpy(dc, c, sizeof(c), cudaMemcpyHostToDevice); cudaMemcpy(dw, w, sizeof(w), cudaMemcpyHostToDevice);
  k_prep<<<1,128>>>(ns, dd, dco, dc, dw, dp, de);
  SegPrep hp[ns]; cudaMemcpy(hp, dp, sizeof(hp), cudaMemcpyDeviceToHost);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  for(int i=0;i<ns;i++){ printf("seg %d deg %d B %.6g S0 %.6g Bq", i, deg[i], hp[i].B, hp[i].S0); for(int q=0;q<8;q++) printf(" %.5g", hp[i].Bq[q]); printf("\n"); }
}
