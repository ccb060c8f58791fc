// FP64 microbenchmarks for the cCG hot-path design on B200 (sm_100a).
// Measures: DADD dependent latency, DMUL->DADD chain step latency,
// DFMA / DMUL+DADD throughput, DMMA (mma.sync f64) throughput, HBM read BW.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_probe fp64_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); std::exit(1);} } while (0)

__global__ void lat_dadd(double* out, long long* cyc, double a, int iters) {
  double acc = a;
  long long t0 = clock64();
  #pragma unroll 1
  for (int i = 0; i < iters; ++i) {
    acc = __dadd_rn(acc, a); acc = __dadd_rn(acc, a); acc = __dadd_rn(acc, a); acc = __dadd_rn(acc, a);
  }
  long long t1 = clock64();
  out[0] = acc; cyc[0] = t1 - t0;
}

// chain step: acc = acc + x[k]*y[k] with products independent of acc
__global__ void lat_chain(const double* x, const double* y, double* out, long long* cyc, int n) {
  double acc = 0.0;
  long long t0 = clock64();
  #pragma unroll 8
  for (int k = 0; k < n; ++k) acc = __dadd_rn(acc, __dmul_rn(x[k], y[k]));
  long long t1 = clock64();
  out[0] = acc; cyc[0] = t1 - t0;
}

template <int CH>
__global__ void tput_mul_add(double* out, double a, double b, int iters) {
  double acc[CH];
  #pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = a + c + threadIdx.x;
  #pragma unroll 1
  for (int i = 0; i < iters; ++i) {
    #pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = __dadd_rn(acc[c], __dmul_rn(acc[c], b));
  }
  double s = 0;
  #pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

template <int CH>
__global__ void tput_fma(double* out, double a, double b, int iters) {
  double acc[CH];
  #pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = a + c + threadIdx.x;
  #pragma unroll 1
  for (int i = 0; i < iters; ++i) {
    #pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = __fma_rn(acc[c], b, a);
  }
  double s = 0;
  #pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

// DMMA m8n8k4: D(8x8) = A(8x4) B(4x8) + C
template <int CH>
__global__ void tput_dmma884(double* out, double a, int iters) {
  double c[CH][2];
  double av = a + threadIdx.x, bv = a - threadIdx.x;
  #pragma unroll
  for (int q = 0; q < CH; ++q) { c[q][0] = 0; c[q][1] = 0; }
  #pragma unroll 1
  for (int i = 0; i < iters; ++i) {
    #pragma unroll
    for (int q = 0; q < CH; ++q)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[q][0]), "+d"(c[q][1]) : "d"(av), "d"(bv));
  }
  double s = 0;
  #pragma unroll
  for (int q = 0; q < CH; ++q) s += c[q][0] + c[q][1];
  if (s == 12345.678) out[0] = s;
}

// DMMA m16n8k16 (sm_90+): A 16x16 (8 regs/thread), B 16x8 (4 regs), C 16x8 (4 regs)
template <int CH>
__global__ void tput_dmma16816(double* out, double a, int iters) {
  double c[CH][4];
  double av[8], bv[4];
  #pragma unroll
  for (int r = 0; r < 8; ++r) av[r] = a + r + threadIdx.x;
  #pragma unroll
  for (int r = 0; r < 4; ++r) bv[r] = a - r - threadIdx.x;
  #pragma unroll
  for (int q = 0; q < CH; ++q) { c[q][0] = c[q][1] = c[q][2] = c[q][3] = 0; }
  #pragma unroll 1
  for (int i = 0; i < iters; ++i) {
    #pragma unroll
    for (int q = 0; q < CH; ++q)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[q][0]), "+d"(c[q][1]), "+d"(c[q][2]), "+d"(c[q][3])
                   : "d"(av[0]), "d"(av[1]), "d"(av[2]), "d"(av[3]), "d"(av[4]), "d"(av[5]), "d"(av[6]), "d"(av[7]),
                     "d"(bv[0]), "d"(bv[1]), "d"(bv[2]), "d"(bv[3]));
  }
  double s = 0;
  #pragma unroll
  for (int q = 0; q < CH; ++q) s += c[q][0] + c[q][1] + c[q][2] + c[q][3];
  if (s == 12345.678) out[0] = s;
}

__global__ void read_bw(const double2* __restrict__ p, size_t n2, double* out) {
  double acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += stride) {
    double2 v = __ldcs(p + i);
    acc += v.x + v.y;
  }
  if (acc == 12345.678) out[0] = acc;
}

static float time_kernel(void (*launch)(void*), void* arg, int reps) {
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  launch(arg); CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(e0));
  for (int r = 0; r < reps; ++r) launch(arg);
  CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
  float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
  return ms / reps;
}

struct Args { double* out; int iters; int grid; int block; const double2* p; size_t n2; };

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int clk_khz = 0; CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
  std::printf("device %s SMs %d L2 %d MB clock(attr) %d MHz\n", prop.name, prop.multiProcessorCount,
              prop.l2CacheSize >> 20, clk_khz / 1000);
  double* out; long long* cyc; CK(cudaMalloc(&out, 64)); CK(cudaMalloc(&cyc, 64));
  // latency
  lat_dadd<<<1, 1>>>(out, cyc, 1.0, 1000); CK(cudaDeviceSynchronize());
  lat_dadd<<<1, 1>>>(out, cyc, 1.0, 10000); CK(cudaDeviceSynchronize());
  long long h; CK(cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost));
  std::printf("DADD dependent latency: %.2f cycles\n", (double)h / 40000.0);
  int n = 1 << 16; double *x, *y; CK(cudaMalloc(&x, n * 8)); CK(cudaMalloc(&y, n * 8));
  CK(cudaMemset(x, 0, n * 8)); CK(cudaMemset(y, 0, n * 8));
  lat_chain<<<1, 1>>>(x, y, out, cyc, n); CK(cudaDeviceSynchronize());
  lat_chain<<<1, 1>>>(x, y, out, cyc, n); CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost));
  std::printf("chain step (ld x,y + DMUL + DADD, L1/L2-hot, 1 thread): %.2f cycles/step\n", (double)h / n);

  const int SM = prop.multiProcessorCount;
  Args a{out, 2000, SM * 8, 256, nullptr, 0};
  auto fl = [](double ms, double lane_ops) { return lane_ops / (ms * 1e-3) / 1e12; };
  {
    float ms = time_kernel([](void* v) { Args* a = (Args*)v; tput_mul_add<8><<<a->grid, a->block>>>(a->out, 1.0, 0.999, a->iters); }, &a, 5);
    double ops = (double)a.grid * a.block * a.iters * 8 * 2;
    std::printf("DMUL+DADD throughput: %.2f T fp64-instr-lanes/s (%.3f ms)\n", fl(ms, ops), ms);
  }
  {
    float ms = time_kernel([](void* v) { Args* a = (Args*)v; tput_fma<8><<<a->grid, a->block>>>(a->out, 1.0, 0.999, a->iters); }, &a, 5);
    double ops = (double)a.grid * a.block * a.iters * 8;
    std::printf("DFMA throughput: %.2f TFLOP/s (%.2f T DFMA lanes/s)\n", 2 * fl(ms, ops), fl(ms, ops));
  }
  {
    float ms = time_kernel([](void* v) { Args* a = (Args*)v; tput_dmma884<4><<<a->grid, a->block>>>(a->out, 1.0, a->iters); }, &a, 5);
    double flops = (double)a.grid * (a.block / 32) * a.iters * 4 * (8 * 8 * 4 * 2);
    std::printf("DMMA m8n8k4 throughput: %.2f TFLOP/s\n", flops / (ms * 1e-3) / 1e12);
  }
  {
    float ms = time_kernel([](void* v) { Args* a = (Args*)v; tput_dmma16816<2><<<a->grid, a->block>>>(a->out, 1.0, a->iters); }, &a, 5);
    double flops = (double)a.grid * (a.block / 32) * a.iters * 2 * (16 * 8 * 16 * 2);
    std::printf("DMMA m16n8k16 throughput: %.2f TFLOP/s\n", flops / (ms * 1e-3) / 1e12);
  }
  {
    size_t bytes = (size_t)4 << 30;
    double2* p; CK(cudaMalloc(&p, bytes)); CK(cudaMemset(p, 0, bytes));
    Args b{out, 0, SM * 4, 512, p, bytes / 16};
    float ms = time_kernel([](void* v) { Args* a = (Args*)v; read_bw<<<a->grid, a->block>>>(a->p, a->n2, a->out); }, &b, 5);
    std::printf("HBM read BW (LDG.128 streaming, 4 GiB): %.1f GB/s\n", bytes / (ms * 1e-3) / 1e9);
    CK(cudaFree(p));
  }
  size_t fr, tot; CK(cudaMemGetInfo(&fr, &tot));
  std::printf("memory free %.1f GB total %.1f GB\n", fr / 1e9, tot / 1e9);
  return 0;
}
