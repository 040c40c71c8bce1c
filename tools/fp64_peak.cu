// fp64_peak.cu — measured FP64 throughput of one B200 (the denominator of the
// limiter's FP64 roofline).  Build + run (tools/fp64_peak.sh):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o fp64_peak fp64_peak.cu
//   ./fp64_peak > profiles/fp64_peak.json
// Each kernel runs kChains independent dependent chains per thread (enough
// ILP x warps to cover the pipe latency) over a grid of 148 x 8 CTAs x 256
// threads, timed with CUDA events (best of 5).  Reported per second:
// DADD / DMUL / DFMA / DMNMX instructions, and IEEE divisions (div.rn.f64:
// MUFU.RCP64H + a DFMA refinement sequence + a slow-path test) and sqrt.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8;
constexpr int kIters = 4096;

template <int kOp>
__global__ void k_fp64(double* out, double seed) {
  double x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = seed + threadIdx.x * 1e-9 + c;
  const double a = 1.0000001, b = 1e-9;
#pragma unroll 4
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      if (kOp == 0) x[c] = x[c] + b;             // DADD
      if (kOp == 1) x[c] = x[c] * a;             // DMUL
      if (kOp == 2) x[c] = __fma_rn(x[c], a, b); // DFMA
      if (kOp == 3) x[c] = fmax(x[c] * 0.5, x[c] - b);  // DMUL + DMNMX (DADD in parallel)
      if (kOp == 4) x[c] = a / x[c];             // IEEE division
      if (kOp == 5) x[c] = sqrt(x[c] + 1.0);     // IEEE sqrt (+ DADD)
    }
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

template <int kOp>
float run(double* out, int blocks) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_fp64<kOp><<<blocks, 256>>>(out, 1.0);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    k_fp64<kOp><<<blocks, 256>>>(out, 1.0 + r);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* out;
  cudaMalloc(&out, 8);
  const int blocks = sms * 8;
  const double ops = (double)blocks * 256 * kIters * kChains;
  const char* names[6] = {"dadd", "dmul", "dfma", "dmul_dmnmx", "ddiv", "dsqrt_dadd"};
  float ms[6];
  ms[0] = run<0>(out, blocks);
  ms[1] = run<1>(out, blocks);
  ms[2] = run<2>(out, blocks);
  ms[3] = run<3>(out, blocks);
  ms[4] = run<4>(out, blocks);
  ms[5] = run<5>(out, blocks);
  printf("{\"device_sms\": %d, \"clock_mhz_attr\": %.0f, \"threads\": %d, \"ops_per_kernel\": %.6g,\n",
         sms, clk / 1e3, blocks * 256, ops);
  printf(" \"note\": \"per second; dmul_dmnmx and dsqrt_dadd count one chain step (2 instructions)\",\n");
  for (int k = 0; k < 6; ++k)
    printf(" \"%s_per_s\": %.6g, \"%s_ms\": %.4f%s\n", names[k], ops / (ms[k] * 1e-3), names[k],
           ms[k], k == 5 ? "" : ",");
  printf("}\n");
  return cudaGetLastError() != cudaSuccess;
}
