// peak.cu -- fp64 roofline denominator: MEASURED_PEAKS.json carries HBM and
// bf16 figures only, so the FP64 peak is measured here with independent DFMA
// chains on every SM (8 chains per thread, no memory traffic).
#include <string>

#include "cbx_device.cuh"
#include "cbx_host.h"

namespace {

__global__ void __launch_bounds__(256) k_dfma(double* out, double a, double b, int iters,
                                              long long* clk) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5,
         x6 = x0 + 6, x7 = x0 + 7;
  const long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
  const double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.678) out[threadIdx.x] = s;  // keep the chains alive
}

}  // namespace

extern "C" CBX_API cbx_status cbx_fp64_peak(int device, double* tflops, double* sm_mhz) {
  using namespace cbx;
  if (cudaSetDevice(device) != cudaSuccess) {
    set_thread_error("cbx_fp64_peak: no such device");
    return CBX_CUDA;
  }
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  double* out;
  long long* clk;
  cudaMalloc(&out, 256 * sizeof(double));
  cudaMalloc(&clk, sizeof(long long));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8, iters = 4096;
  k_dfma<<<blocks, 256>>>(out, 0.999999, 1e-7, 64, clk);  // warm-up
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    k_dfma<<<blocks, 256>>>(out, 0.999999, 1e-7, iters, clk);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  long long cycles = 0;
  cudaMemcpy(&cycles, clk, sizeof cycles, cudaMemcpyDeviceToHost);
  const double flops = 2.0 * 8 * 16 * (double)iters * blocks * 256;
  *tflops = flops / (best * 1e-3) / 1e12;
  // the timed block ran for `cycles` SM clocks; blocks run in waves of
  // (resident blocks), so the clock estimate is cycles * waves / time
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dfma, 256, 0);
  const double waves = (double)blocks / ((double)sms * (per_sm > 0 ? per_sm : 1));
  if (sm_mhz) *sm_mhz = (double)cycles * (waves < 1 ? 1 : waves) / (best * 1e-3) / 1e6;
  cudaFree(out);
  cudaFree(clk);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_thread_error(std::string("cbx_fp64_peak: ") + cudaGetErrorString(e));
    return CBX_CUDA;
  }
  return CBX_OK;
}
