// fold_bench.cu — cycles of one sequential fold acc = ((0 + d0) + d1) + ... of
// nb doubles held in shared memory, by one lane (the PARITY block_dot chain,
// pcg.hpp:37-44), for several load schedules. Sizes pcg_kernel_h8p's fold.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a --fmad=false -o fold_bench tools/fold_bench.cu && ./fold_bench
#include <cstdio>

__device__ __noinline__ double fold_blocks16(const double* seg, int nb) {  // h8p's current schedule
  const int nfull = nb & ~15;
  double tail[15];
#pragma unroll
  for (int t = 0; t < 15; ++t) tail[t] = nfull + t < nb ? seg[nfull + t] : 0.0;
  double cur[16];
#pragma unroll
  for (int t = 0; t < 16; ++t) cur[t] = nfull > 0 ? seg[t] : 0.0;
  double acc = 0.0;
  for (int k = 0; k < nfull; k += 16) {
    const int kn = k + 16 < nfull ? k + 16 : k;
    double nxt[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) nxt[t] = seg[kn + t];
#pragma unroll
    for (int t = 0; t < 16; ++t) acc = acc + cur[t];
#pragma unroll
    for (int t = 0; t < 16; ++t) cur[t] = nxt[t];
  }
#pragma unroll
  for (int t = 0; t < 15; ++t)
    if (nfull + t < nb) acc = acc + tail[t];
  return acc;
}

__device__ __noinline__ double fold_simple(const double* seg, int nb) {
  double acc = 0.0;
#pragma unroll 8
  for (int k = 0; k < nb; ++k) acc = acc + seg[k];
  return acc;
}

// all loads first into a register file of 128 (fixed trip, nb <= 128), then
// the adds; the trailing adds beyond nb are skipped by a computed jump (switch)
__device__ __noinline__ double fold_regs(const double* seg, int nb) {
  double v[128];
#pragma unroll
  for (int t = 0; t < 128; ++t) v[t] = seg[t];
  double acc = 0.0;
#pragma unroll
  for (int t = 0; t < 128; ++t) {
    if (t >= nb) break;
    acc = acc + v[t];
  }
  return acc;
}

// the warp's lanes hold 4 values each (lane l: seg[l], seg[32 + l], ...); lane 0 folds via shuffles
__device__ __noinline__ double fold_shfl(const double* seg, int nb) {
  const int lane = threadIdx.x & 31;
  double v[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) v[r] = seg[32 * r + lane];
  double acc = 0.0;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
#pragma unroll
    for (int l = 0; l < 32; ++l) {
      const double x = __shfl_sync(0xffffffffu, v[r], l);
      if (32 * r + l < nb) acc = acc + x;
    }
  }
  return acc;
}

// front-padded with +0.0 to a multiple of 16 (exact: the fold starts from
// 0.0 anyway and 0.0 + 0.0 = +0.0), ping-pong register blocks, no per-element
// control flow: the adds run back to back at the DADD latency
__device__ __noinline__ double fold_padded(const double* seg, int nb) {
  const int pad = (16 - (nb & 15)) & 15, total = nb + pad;
  auto ld = [&](int k) { return k >= pad && k < total ? seg[k - pad] : 0.0; };
  double A[16], Bv[16], acc = 0.0;
#pragma unroll
  for (int t = 0; t < 16; ++t) A[t] = ld(t);
  for (int k = 0; k < total; k += 32) {
#pragma unroll
    for (int t = 0; t < 16; ++t) Bv[t] = ld(k + 16 + t);
#pragma unroll
    for (int t = 0; t < 16; ++t) acc = acc + A[t];
    if (k + 16 >= total) break;
#pragma unroll
    for (int t = 0; t < 16; ++t) A[t] = ld(k + 32 + t);
#pragma unroll
    for (int t = 0; t < 16; ++t) acc = acc + Bv[t];
  }
  return acc;
}

// front-padded, the loads as one inline-PTX block ahead of the adds (56
// ld.shared.v2.f64 into registers), then 112 dependent add.rn.f64
// padded, every load issued up front through a volatile pointer, then the
// dependent adds (16-value blocks, no per-element predicates)
__device__ __noinline__ double fold_vol(const double* seg0, int nb) {
  const int pad = (16 - (nb & 15)) & 15, total = nb + pad;
  const volatile double* base = seg0 + 16 - pad;
  double v[112];
#pragma unroll
  for (int t = 0; t < 112; ++t) v[t] = base[t];
  double acc = 0.0;
#pragma unroll
  for (int b = 0; b < 7; ++b) {
    if (16 * b >= total) break;
#pragma unroll
    for (int t = 0; t < 16; ++t) acc = acc + v[16 * b + t];
  }
  return acc;
}

__device__ __forceinline__ double2 lds2(const double* p) {
  double2 r;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "r"(static_cast<unsigned>(__cvta_generic_to_shared(p))));
  return r;
}
__device__ __noinline__ double fold_asm(const double* seg0, int nb) {
  // seg0 has 16 leading zeros: element k of the padded sequence is seg0[16 - pad + k]
  const int pad = (16 - (nb & 15)) & 15, total = nb + pad;
  const double* base = seg0 + 16 - pad;  // may be 8-byte aligned only: scalar loads for odd pad
  double v[112];
  if ((pad & 1) == 0) {
#pragma unroll
    for (int t = 0; t < 56; ++t) {
      const double2 q = lds2(base + 2 * t);
      v[2 * t] = q.x, v[2 * t + 1] = q.y;
    }
  } else {
#pragma unroll
    for (int t = 0; t < 112; ++t) asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v[t]) : "r"(static_cast<unsigned>(__cvta_generic_to_shared(base + t))));
  }
  double acc = 0.0;
#pragma unroll
  for (int t = 0; t < 112; ++t)
    if (t < total) acc = acc + v[t];
  return acc;
}

__global__ void bench(double* out, long long* cyc, int nb, int reps) {
  __shared__ double seg[128];
  __shared__ __align__(16) double seg0[16 + 128];
  for (int k = threadIdx.x; k < 128; k += blockDim.x) seg[k] = 1.0 + 1e-3 * k;
  for (int k = threadIdx.x; k < 144; k += blockDim.x) seg0[k] = k < 16 ? 0.0 : 1.0 + 1e-3 * (k - 16);
  __syncthreads();
  double s = 0;
  long long t[7];
  t[0] = clock64();
  for (int r = 0; r < reps; ++r) s += (threadIdx.x == 0) ? fold_blocks16(seg, nb) : 0.0;
  t[1] = clock64();
  for (int r = 0; r < reps; ++r) s += (threadIdx.x == 0) ? fold_simple(seg, nb) : 0.0;
  t[2] = clock64();
  for (int r = 0; r < reps; ++r) s += (threadIdx.x == 0) ? fold_regs(seg, nb) : 0.0;
  t[3] = clock64();
  for (int r = 0; r < reps; ++r) s += fold_shfl(seg, nb);
  t[4] = clock64();
  for (int r = 0; r < reps; ++r) s += (threadIdx.x == 0) ? fold_padded(seg, nb) : 0.0;
  t[5] = clock64();
  for (int r = 0; r < reps; ++r) s += (threadIdx.x == 0) ? fold_vol(seg0, nb) : 0.0;
  t[6] = clock64();
  if (threadIdx.x == 0 && fold_vol(seg0, nb) != fold_simple(seg, nb)) printf("VOL MISMATCH nb %d\n", nb);
  if (threadIdx.x == 0 && fold_padded(seg, nb) != fold_simple(seg, nb)) printf("MISMATCH nb %d\n", nb);
  out[threadIdx.x] = s;
  if (threadIdx.x == 0)
    for (int k = 0; k < 6; ++k) cyc[k] = t[k + 1] - t[k];
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 32 * 8);
  cudaMallocManaged(&cyc, 6 * 8);
  const int reps = 200;
  for (int nb : {101, 112, 64, 17, 1}) {
    bench<<<1, 32>>>(out, cyc, nb, reps);
    cudaDeviceSynchronize();
    printf("nb %3d: blocks16 %.0f  simple %.0f  regs %.0f  shfl %.0f  padded %.0f  vol %.0f cycles per fold (pure chain ~%.0f)\n",
           nb, cyc[0] / double(reps), cyc[1] / double(reps), cyc[2] / double(reps), cyc[3] / double(reps),
           cyc[4] / double(reps), cyc[5] / double(reps), 8.19 * nb);
  }
  return 0;
}
