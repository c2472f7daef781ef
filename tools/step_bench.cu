// Per-pivot-step latency floor for a 128-thread CTA: barrier + broadcast,
// + rsqrt, + rank-1 patch update (2x4 and 4x8 patches).
#include <cstdio>
template <int V, int NR, int NC>
__global__ void k(double* out, long long* cyc) {
  __shared__ double buf[2][128];
  const int t = threadIdx.x;
  double a[NR][NC];
  for (int i = 0; i < NR; ++i) for (int j = 0; j < NC; ++j) a[i][j] = 1.0 + t * 1e-3 + i + j;
  long long t0 = clock64();
  for (int s = 0; s < 256; ++s) {
    double* b = buf[s & 1];
    if ((t & 7) == ((s >> 2) & 7)) { b[(t >> 3) * 2] = a[0][0]; b[(t >> 3) * 2 + 1] = a[NR - 1][0]; }
    __syncthreads();
    double piv = b[s & 63] + 2.0;
    double inv = V >= 2 ? rsqrt(piv) : piv;
    if (V >= 3) {
      double li[NR], lk[NC];
      for (int i = 0; i < NR; ++i) li[i] = b[(t + i) & 63] * inv;
      for (int j = 0; j < NC; ++j) lk[j] = b[(t * 3 + j) & 63] * inv;
      for (int i = 0; i < NR; ++i) for (int j = 0; j < NC; ++j) a[i][j] = fma(-li[i] * 1e-9, lk[j], a[i][j]);
    } else {
      a[0][0] += inv * 1e-9;
    }
  }
  long long t1 = clock64();
  double sacc = 0; for (int i = 0; i < NR; ++i) for (int j = 0; j < NC; ++j) sacc += a[i][j];
  out[t] = sacc;
  if (t == 0) cyc[0] = (t1 - t0) / 256;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 4096); cudaMalloc(&c, 8); long long h;
#define RUN(V, NR, NC) k<V, NR, NC><<<1, 128>>>(o, c); k<V, NR, NC><<<1, 128>>>(o, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("{\"variant\": %d, \"patch\": \"%dx%d\", \"cycles_per_step\": %lld}\n", V, NR, NC, h);
  RUN(1, 2, 4) RUN(2, 2, 4) RUN(3, 2, 4) RUN(3, 4, 8) RUN(3, 1, 2)
  return 0;
}
