// dependent fp64 add chain latency (cycles per __dadd_rn) on one warp
#include <cstdio>
__global__ void chain(double* out, double a, int n, long long* cyc) {
  double x = a, y = a * 0.5;
  long long t0 = clock64();
  for (int i = 0; i < n; i++) {
    x = __dadd_rn(x, y);
    x = __dadd_rn(x, y);
    x = __dadd_rn(x, y);
    x = __dadd_rn(x, y);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { *out = x; *cyc = t1 - t0; }
}
__global__ void chainf(float* out, float a, int n, long long* cyc) {
  float x = a, y = a * 0.5f;
  long long t0 = clock64();
  for (int i = 0; i < n; i++) {
    x = __fadd_rn(x, y);
    x = __fadd_rn(x, y);
    x = __fadd_rn(x, y);
    x = __fadd_rn(x, y);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { *out = x; *cyc = t1 - t0; }
}
int main() {
  double* d; float* f; long long* c; long long h;
  cudaMalloc(&d, 8); cudaMalloc(&f, 4); cudaMalloc(&c, 8);
  const int n = 1 << 16;
  for (int rep = 0; rep < 2; rep++) {
    chain<<<1, 32>>>(d, 1.0, n, c);
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("DADD dependent latency: %.2f cycles\n", (double)h / (4.0 * n));
    chainf<<<1, 32>>>(f, 1.0f, n, c);
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("FADD dependent latency: %.2f cycles\n", (double)h / (4.0 * n));
  }
  return 0;
}
