// Microbenchmark: dependent-chain latency of DMUL / DADD / DFMA and the
// single-warp throughput of the walk recurrence on this GPU (clock64).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(int n, double a, double* out, long long* cyc) {
  double x = a, y = a + 1.0, z = a * 0.5;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = x * 0.9999999;
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) y = y + 1e-9;
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) z = fma(z, 0.9999999, 1e-12);
  long long t3 = clock64();
  out[threadIdx.x] = x + y + z;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; }
}

// the walk's node recurrence, one warp
__global__ void walk(int n, const double* v, double* out, long long* cyc) {
  double pdf = 0.3 + threadIdx.x * 1e-6, ratio = 0.99999, q = 0.9999999, acc0 = 0, acc1 = 0, acc2 = 0, h = 0.025;
  long long t0 = clock64();
#pragma unroll 4
  for (int j = 0; j < n; ++j) {
    double wp = h * pdf; double vj = v[j & 1023];
    acc0 += wp; double wv = wp * vj; acc1 += wv; acc2 += wv * vj; pdf *= ratio; ratio *= q;
  }
  long long t1 = clock64();
  out[threadIdx.x] = acc0 + acc1 + acc2 + pdf;
  if (threadIdx.x == 0) cyc[3] = t1 - t0;
}

// software-pipelined: the pdf/ratio chain of group g+1 runs ahead of the
// accumulation of group g (same products in the same order)
__global__ void walk_sp(int n, const double* v, double* out, long long* cyc) {
  double pdf = 0.3 + threadIdx.x * 1e-6, ratio = 0.99999, q = 0.9999999, acc0 = 0, acc1 = 0, acc2 = 0, h = 0.025;
  long long t0 = clock64();
  double p0 = pdf, p1, p2, p3;
  p1 = p0 * ratio; ratio *= q; p2 = p1 * ratio; ratio *= q; p3 = p2 * ratio; ratio *= q;
  pdf = p3 * ratio; ratio *= q;  // pdf of the next group's first node
  for (int j = 0; j < n; j += 4) {
    double n0 = pdf, n1, n2, n3, r = ratio;
    n1 = n0 * r; r *= q; n2 = n1 * r; r *= q; n3 = n2 * r; r *= q;
    double nn = n3 * r; r *= q;
    double v0 = v[j & 1023], v1 = v[(j + 1) & 1023], v2 = v[(j + 2) & 1023], v3 = v[(j + 3) & 1023];
    double w0 = h * p0; acc0 += w0; double x0 = w0 * v0; acc1 += x0; acc2 += x0 * v0;
    double w1 = h * p1; acc0 += w1; double x1 = w1 * v1; acc1 += x1; acc2 += x1 * v1;
    double w2 = h * p2; acc0 += w2; double x2 = w2 * v2; acc1 += x2; acc2 += x2 * v2;
    double w3 = h * p3; acc0 += w3; double x3 = w3 * v3; acc1 += x3; acc2 += x3 * v3;
    p0 = n0; p1 = n1; p2 = n2; p3 = n3; pdf = nn; ratio = r;
  }
  long long t1 = clock64();
  out[threadIdx.x] = acc0 + acc1 + acc2 + pdf;
  if (threadIdx.x == 0) cyc[4] = t1 - t0;
}

// two independent walks per thread
__global__ void walk2(int n, const double* v, double* out, long long* cyc) {
  double pa = 0.3 + threadIdx.x * 1e-6, ra = 0.99999, pb = 0.31, rb = 0.99998, q = 0.9999999, h = 0.025;
  double a0 = 0, a1 = 0, a2 = 0, b0 = 0, b1 = 0, b2 = 0;
  long long t0 = clock64();
#pragma unroll 4
  for (int j = 0; j < n; ++j) {
    double vj = v[j & 1023];
    double wa = h * pa; a0 += wa; double xa = wa * vj; a1 += xa; a2 += xa * vj; pa *= ra; ra *= q;
    double wb = h * pb; b0 += wb; double xb = wb * vj; b1 += xb; b2 += xb * vj; pb *= rb; rb *= q;
  }
  long long t1 = clock64();
  out[threadIdx.x] = a0 + a1 + a2 + b0 + b1 + b2 + pa + pb;
  if (threadIdx.x == 0) cyc[5] = t1 - t0;
}

int main() {
  double *out, *v; long long* cyc;
  cudaMalloc(&out, 1024 * 8); cudaMalloc(&v, 1024 * 8); cudaMallocManaged(&cyc, 8 * 8);
  cudaMemset(v, 0, 1024 * 8);
  const int n = 1 << 16;
  lat<<<1, 32>>>(n, 1.0, out, cyc); cudaDeviceSynchronize();
  lat<<<1, 32>>>(n, 1.0, out, cyc); cudaDeviceSynchronize();
  printf("latency cycles: DMUL %.2f  DADD %.2f  DFMA %.2f\n", cyc[0] / (double)n, cyc[1] / (double)n, cyc[2] / (double)n);
  for (int warps = 1; warps <= 32; warps *= 2) {
    walk<<<1, 32 * warps>>>(n, v, out, cyc); cudaDeviceSynchronize();
    walk<<<1, 32 * warps>>>(n, v, out, cyc); cudaDeviceSynchronize();
    printf("walk: %2d warps/CTA (1 SM): %.2f cycles per node per warp\n", warps, cyc[3] / (double)n);
  }
  for (int warps = 1; warps <= 32; warps *= 2) {
    walk_sp<<<1, 32 * warps>>>(n, v, out, cyc); cudaDeviceSynchronize();
    walk_sp<<<1, 32 * warps>>>(n, v, out, cyc); cudaDeviceSynchronize();
    walk2<<<1, 32 * warps>>>(n, v, out, cyc); cudaDeviceSynchronize();
    walk2<<<1, 32 * warps>>>(n, v, out, cyc); cudaDeviceSynchronize();
    printf("walk_sp: %2d warps: %.2f cyc/node/warp | walk2 (2 walks/thread): %.2f cyc per node-pair/warp\n",
           warps, cyc[4] / (double)n, cyc[5] / (double)n);
  }
  return 0;
}
