// fp64_lat.cu — dependent-chain latency of DADD / DMUL / DFMA and of a
// shared-memory load + DADD chain on one warp (clock64), plus DADD issue
// throughput with 16 independent chains per thread. Sizes the PARITY block_dot
// fold (a 101-long sequential DADD chain at C3).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o fp64_lat tools/fp64_lat.cu && ./fp64_lat
#include <cstdio>

__global__ void lat(double* out, long long* cyc, double a, double b, int n) {
  __shared__ double sm[256];
  for (int k = threadIdx.x; k < 256; k += blockDim.x) sm[k] = 1e-3 * k;
  __syncthreads();
  double x = a, y = a, z = a, w = 0.0;
  long long t0 = clock64();
#pragma unroll 1
  for (int k = 0; k < n; ++k) {
#pragma unroll
    for (int j = 0; j < 16; ++j) x = x + b;
  }
  long long t1 = clock64();
#pragma unroll 1
  for (int k = 0; k < n; ++k) {
#pragma unroll
    for (int j = 0; j < 16; ++j) y = y * b;
  }
  long long t2 = clock64();
#pragma unroll 1
  for (int k = 0; k < n; ++k) {
#pragma unroll
    for (int j = 0; j < 16; ++j) z = fma(z, b, a);
  }
  long long t3 = clock64();
  // sequential fold over shared-memory values (loads independent of the chain)
#pragma unroll 1
  for (int k = 0; k < n; ++k) {
#pragma unroll
    for (int j = 0; j < 16; ++j) w = w + sm[(k * 16 + j) & 255];
  }
  long long t4 = clock64();
  double c[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) c[j] = a + j;
#pragma unroll 1
  for (int k = 0; k < n; ++k) {
#pragma unroll
    for (int j = 0; j < 16; ++j) c[j] = c[j] + b;
  }
  long long t5 = clock64();
  double s = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) s += c[j];
  out[threadIdx.x] = x + y + z + w + s;
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
    cyc[2] = t3 - t2;
    cyc[3] = t4 - t3;
    cyc[4] = t5 - t4;
  }
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * 8);
  cudaMallocManaged(&cyc, 8 * 8);
  const int n = 1000;
  for (int warps : {1, 4}) {
    lat<<<1, 32 * warps>>>(out, cyc, 1.0, 1.0000001, n);
    cudaDeviceSynchronize();
    const double ops = 16.0 * n;
    printf("warps/CTA %d: DADD %.2f  DMUL %.2f  DFMA %.2f  LDS+DADD fold %.2f cycles/op (dependent);"
           " 16 independent DADD chains: %.2f cycles per warp-instruction\n",
           warps, cyc[0] / ops, cyc[1] / ops, cyc[2] / ops, cyc[3] / ops, cyc[4] / (ops * 16));
  }
  return 0;
}
