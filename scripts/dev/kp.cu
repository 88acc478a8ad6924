
#include <cstdio>
#include <cstdint>
#include <cmath>
struct SegPrep { double B, S0; double Bq[8]; };
// Exact binomial coefficients C(n,k), n <= 10.
__constant__ double c_binom[11][11] = {
    {1}, {1, 1}, {1, 2, 1}, {1, 3, 3, 1}, {1, 4, 6, 4, 1}, {1, 5, 10, 10, 5, 1}, {1, 6, 15, 20, 15, 6, 1},
    {1, 7, 21, 35, 35, 21, 7, 1}, {1, 8, 28, 56, 70, 56, 28, 8, 1}, {1, 9, 36, 84, 126, 126, 84, 36, 9, 1},
    {1, 10, 45, 120, 210, 252, 210, 120, 45, 10, 1}};

// Bounds on homogeneous control points (X_i, Y_i, W_i) = w_i (x_i, y_i, 1),
// i = 0..N, held in registers (templated on the degree, fully unrolled).
// Written without accumulating into local arrays (an earlier version of that
// shape was miscompiled by nvcc 12.9 -O3 on sm_100a: scripts/dev/kp.cu).
//
// Hodograph-numerator Bernstein bound: |gamma'| = |X'W - XW'| / W^2 with
//   X'W - XW' = N sum_k D_k B_k^{2N-1},
//   D_k = sum_{i+j=k} C(N-1,i)C(N,j)/C(2N-1,k) [W_j (X_{i+1}-X_i) - (W_{i+1}-W_i) X_j],
//   W^2 = sum_k E_k B_k^{2N},  E_k = sum_{i+j=k} C(N,i)C(N,j)/C(2N,k) W_i W_j,
// so |gamma'| <= N max_k |D_k| / min_k E_k (convex-hull property).
template <int N>
__device__ __forceinline__ double hodo_bound(const double (&X)[N + 1], const double (&Y)[N + 1],
                                             const double (&W)[N + 1]) {
  double dmax = 0.0, emin = INFINITY;
#pragma unroll
  for (int k = 0; k <= 2 * N - 1; ++k) {
    double dx = 0.0, dy = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const int j = k - i;
      if (j < 0 || j > N) continue;
      const double c = c_binom[N - 1][i] * c_binom[N][j] / c_binom[2 * N - 1][k];
      dx += c * (W[j] * (X[i + 1] - X[i]) - (W[i + 1] - W[i]) * X[j]);
      dy += c * (W[j] * (Y[i + 1] - Y[i]) - (W[i + 1] - W[i]) * Y[j]);
    }
    dmax = fmax(dmax, hypot(dx, dy));
  }
#pragma unroll
  for (int k = 0; k <= 2 * N; ++k) {
    double e = 0.0;
#pragma unroll
    for (int i = 0; i <= N; ++i) {
      const int j = k - i;
      if (j < 0 || j > N) continue;
      e += c_binom[N][i] * c_binom[N][j] / c_binom[2 * N][k] * W[i] * W[j];
    }
    emin = fmin(emin, e);
  }
  return N * dmax / emin;
}

template <int N>
__device__ __forceinline__ double floater_bound(const double (&X)[N + 1], const double (&Y)[N + 1],
                                                const double (&W)[N + 1]) {
  double wmax = W[0], wmin = W[0], dmax = 0.0, diam = 0.0;
#pragma unroll
  for (int i = 1; i <= N; ++i) { wmax = fmax(wmax, W[i]); wmin = fmin(wmin, W[i]); }
#pragma unroll
  for (int i = 0; i <= N; ++i)
#pragma unroll
    for (int j = i + 1; j <= N; ++j) {
      const double l = hypot(X[j] / W[j] - X[i] / W[i], Y[j] / W[j] - Y[i] / W[i]);
      diam = fmax(diam, l);
      if (j == i + 1) dmax = fmax(dmax, l);
    }
  if (wmax == wmin) return N * dmax;
  const double r = wmax / wmin;
  return fmin(N * r * diam, N * r * r * dmax);
}

// piece [q/8,(q+1)/8]: three de Casteljau halvings along the bits of q
template <int N>
__device__ __forceinline__ void dyadic_piece(const double (&X)[N + 1], const double (&Y)[N + 1],
                                             const double (&W)[N + 1], int q, double (&a)[N + 1],
                                             double (&b)[N + 1], double (&c)[N + 1]) {
#pragma unroll
  for (int i = 0; i <= N; ++i) { a[i] = X[i]; b[i] = Y[i]; c[i] = W[i]; }
#pragma unroll
  for (int lvl = 2; lvl >= 0; --lvl) {
    const bool right = (q >> lvl) & 1;
    double ta[N + 1], tb[N + 1], tc[N + 1];
#pragma unroll
    for (int i = 0; i <= N; ++i) { ta[i] = a[i]; tb[i] = b[i]; tc[i] = c[i]; }
    // after round r, entry 0 is the left half's point r, entry N-r the right half's
#pragma unroll
    for (int r = 1; r <= N; ++r) {
#pragma unroll
      for (int j = 0; j <= N - r; ++j) {
        ta[j] = 0.5 * (ta[j] + ta[j + 1]);
        tb[j] = 0.5 * (tb[j] + tb[j + 1]);
        tc[j] = 0.5 * (tc[j] + tc[j + 1]);
      }
      if (right) {
        a[N - r] = ta[N - r]; b[N - r] = tb[N - r]; c[N - r] = tc[N - r];
      } else {
        a[r] = ta[0]; b[r] = tb[0]; c[r] = tc[0];
      }
    }
  }
}

template <int N>
__device__ __forceinline__ void prep_n(const double *__restrict__ ctrl, const double *__restrict__ w, int o,
                                       SegPrep *__restrict__ out, uint8_t *__restrict__ err_out) {
  double X[N + 1], Y[N + 1], W[N + 1];
  bool err = false;
  double lpoly = 0.0;
#pragma unroll
  for (int j = 0; j <= N; ++j) {
    const double x = ctrl[2 * (o + j)], y = ctrl[2 * (o + j) + 1], wj = w ? w[o + j] : 1.0;
    err |= !isfinite(x) || !isfinite(y) || !isfinite(wj) || !(wj > 0.0);
    X[j] = wj * x; Y[j] = wj * y; W[j] = wj;
    if (j) lpoly += hypot(x - ctrl[2 * (o + j - 1)], y - ctrl[2 * (o + j - 1) + 1]);
  }
  *err_out = err ? 1 : 0;
  if (err) {
    out->B = out->S0 = 0.0;
    for (int q = 0; q < 8; ++q) out->Bq[q] = 0.0;
    return;
  }
  const double B = fmin(floater_bound<N>(X, Y, W), hodo_bound<N>(X, Y, W));
  out->B = B;
  out->S0 = fmin(B, lpoly);
#pragma unroll 1
  for (int q = 0; q < 8; ++q) {
    double a[N + 1], b[N + 1], c[N + 1];
    dyadic_piece<N>(X, Y, W, q, a, b, c);
    out->Bq[q] = fmin(B, 8.0 * hodo_bound<N>(a, b, c));
  }
}

__global__ void k_prep(int32_t n_segs, const int32_t *__restrict__ deg, const int32_t *__restrict__ coff,
                       const double *__restrict__ ctrl, const double *__restrict__ w,
                       SegPrep *__restrict__ prep, uint8_t *__restrict__ serr) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_segs) return;
  const int o = coff[s];
  switch (deg[s]) {
    case 1: prep_n<1>(ctrl, w, o, prep + s, serr + s); break;
    case 2: prep_n<2>(ctrl, w, o, prep + s, serr + s); break;
    case 3: prep_n<3>(ctrl, w, o, prep + s, serr + s); break;
    case 4: prep_n<4>(ctrl, w, o, prep + s, serr + s); break;
    default: prep_n<5>(ctrl, w, o, prep + s, serr + s); break;
  }
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
