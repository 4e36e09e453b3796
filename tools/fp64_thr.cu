// fp64_thr.cu — FP64 issue throughput of one SM: W warps, each thread running
// 8 independent DADD (or DMUL, or DADD+DMUL pairs) chains. Prints cycles per
// warp-instruction per SM sub-partition (SMSP), which sizes the matvec phases
// of the PARITY kernels (every product term is a DMUL and a DADD: no FMA).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a --fmad=false -o fp64_thr tools/fp64_thr.cu && ./fp64_thr
#include <cstdio>

template <int KIND>
__global__ void thr(double* out, long long* cyc, double y, int n) {
  double a[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) a[c] = threadIdx.x * 1e-3 + c;
  __syncthreads();
  const long long t0 = clock64();
  for (int k = 0; k < n; ++k) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (KIND == 0) a[c] = a[c] + y;
      if (KIND == 1) a[c] = a[c] * y;
      if (KIND == 2) a[c] = a[c] + a[c] * y;  // DMUL then dependent DADD (a product term)
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += a[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * 8);
  cudaMallocManaged(&cyc, 8);
  const int n = 4096;
  const char* names[3] = {"DADD", "DMUL", "DMUL+DADD"};
  for (int kind = 0; kind < 3; ++kind)
    for (int warps : {1, 2, 4, 8, 16, 32}) {
      auto k = kind == 0 ? thr<0> : kind == 1 ? thr<1> : thr<2>;
      k<<<1, 32 * warps>>>(out, cyc, 1.0000001, n);
      cudaDeviceSynchronize();
      const double instr = double(n) * 8 * (kind == 2 ? 2 : 1) * warps;  // warp-instructions in the SM
      const int smsp = warps < 4 ? warps : 4;
      printf("%-10s warps %2d: %.3f cycles per warp-instruction per SMSP\n", names[kind], warps,
             cyc[0] / (instr / smsp));
    }
  return 0;
}
