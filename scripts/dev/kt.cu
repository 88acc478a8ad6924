
#include <cstdio>
#include <cmath>
__device__ __forceinline__ double binomd(int n, int k) {
  // exact small binomials (n <= 10)
  const double f[11] = {1, 1, 2, 6, 24, 120, 720, 5040, 40320, 362880, 3628800};
  return f[n] / (f[k] * f[n - k]);
}

// H: flat homogeneous control points, H[3i+0..2] = (w x, w y, w), i = 0..n.
// Returns max_k |D_k| / min_k E_k (hodograph numerator over W^2, Bernstein form).
__device__ __forceinline__ double hodo_bound(int n, const double *H) {
  double Dx[10], Dy[10], E[11];
#pragma unroll
  for (int k = 0; k < 10; ++k) { Dx[k] = 0.0; Dy[k] = 0.0; }
#pragma unroll
  for (int k = 0; k < 11; ++k) E[k] = 0.0;
  for (int i = 0; i < n; ++i) {
    const double wi = H[3 * i + 2], wi1 = H[3 * (i + 1) + 2];
    const double xi = H[3 * i] / wi, yi = H[3 * i + 1] / wi;
    const double xi1 = H[3 * (i + 1)] / wi1, yi1 = H[3 * (i + 1) + 1] / wi1;
    for (int j = 0; j <= n; ++j) {
      const double wj = H[3 * j + 2], xj = H[3 * j] / wj, yj = H[3 * j + 1] / wj;
      const double c = binomd(n - 1, i) * binomd(n, j) / binomd(2 * n - 1, i + j) * wj;
      Dx[i + j] += c * (wi1 * (xi1 - xj) - wi * (xi - xj));
      Dy[i + j] += c * (wi1 * (yi1 - yj) - wi * (yi - yj));
    }
  }
  for (int i = 0; i <= n; ++i)
    for (int j = 0; j <= n; ++j)
      E[i + j] += binomd(n, i) * binomd(n, j) / binomd(2 * n, i + j) * H[3 * i + 2] * H[3 * j + 2];
  double dmax = 0.0, emin = INFINITY;
  for (int k = 0; k <= 2 * n - 1; ++k) dmax = fmax(dmax, hypot(Dx[k], Dy[k]));
  for (int k = 0; k <= 2 * n; ++k) emin = fmin(emin, E[k]);
  return n * dmax / emin;
}

__device__ __forceinline__ double floater_bound(int n, const double *H) {
  double wmax = 0.0, wmin = INFINITY, dmax = 0.0, diam = 0.0;
  for (int i = 0; i <= n; ++i) { wmax = fmax(wmax, H[3 * i + 2]); wmin = fmin(wmin, H[3 * i + 2]); }
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

// de Casteljau split at 1/2 of the flat homogeneous control points (in place:
// H becomes the left half, R receives the right half)
__device__ __forceinline__ void hsplit_half(int n, double *H, double *R) {
  double T[18];
  for (int i = 0; i < 3 * (n + 1); ++i) T[i] = H[i];
  for (int c = 0; c < 3; ++c) R[3 * n + c] = T[3 * n + c];
  for (int r = 1; r <= n; ++r) {
    for (int j = 0; j <= n - r; ++j)
      for (int c = 0; c < 3; ++c) T[3 * j + c] = 0.5 * (T[3 * j + c] + T[3 * (j + 1) + c]);
    for (int c = 0; c < 3; ++c) { H[3 * r + c] = T[c]; R[3 * (n - r) + c] = T[3 * (n - r) + c]; }
  }
}


__global__ void kt() {
  double P[3][2]={{1,0},{1,1},{0,1}}; double w[3]={1,0.70710678118654752,1}; int n=2;
  double H[18]; for(int i=0;i<=n;i++){H[3*i]=w[i]*P[i][0];H[3*i+1]=w[i]*P[i][1];H[3*i+2]=w[i];}
  printf("full hodo %.10g floater %.10g\n", hodo_bound(n,H), floater_bound(n,H));
  for(int q=0;q<8;q++){ double A[18],Rr[18]; for(int i=0;i<3*(n+1);i++)A[i]=H[i];
    for(int lvl=2;lvl>=0;--lvl){ hsplit_half(n,A,Rr); if((q>>lvl)&1) for(int i=0;i<3*(n+1);i++)A[i]=Rr[i]; }
    printf("piece %d hodo %.10g floater %.10g  A0 %g %g %g A1 %g %g %g A2 %g %g %g\n", q, 8*hodo_bound(n,A), 8*floater_bound(n,A), A[0],A[1],A[2],A[3],A[4],A[5],A[6],A[7],A[8]); }
}
int main(){ kt<<<1,1>>>(); cudaDeviceSynchronize(); printf("err %s\n", cudaGetErrorString(cudaGetLastError())); }
