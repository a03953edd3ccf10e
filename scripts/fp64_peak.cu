// fp64 ceilings of this B200: DFMA, DADD, DMUL issue
// throughput and the correctly rounded division sequence the stencil uses
// (__drcp_rn + two Markstein corrections), each with 8 independent chains per
// thread on a full persistent grid.  Prints one JSON line per op.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CH = 8;

template <int OP>
__global__ void __launch_bounds__(256) kern(double* out, int iters, double a, double b) {
  double x[CH];
#pragma unroll
  for (int k = 0; k < CH; ++k) x[k] = 1.0 + 1e-3 * (threadIdx.x + k);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      if (OP == 0) x[k] = __fma_rn(x[k], a, b);
      else if (OP == 1) x[k] = __dadd_rn(x[k], b);
      else if (OP == 2) x[k] = __dmul_rn(x[k], a);
      else {  // a / x[k], correctly rounded: rcp + two corrections
        const double r = __drcp_rn(x[k]);
        double q = __dmul_rn(a, r);
        double e = __fma_rn(-x[k], q, a);
        q = __fma_rn(e, r, q);
        e = __fma_rn(-x[k], q, a);
        x[k] = __fma_rn(e, r, q) + 1.0;
      }
    }
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < CH; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;
}

template <int OP>
double run(int blocks, int iters, float* ms_out) {
  double* out;
  cudaMalloc(&out, 8);
  kern<OP><<<blocks, 256>>>(out, 100, 1.0000001, 1e-9);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    kern<OP><<<blocks, 256>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaFree(out);
  *ms_out = best;
  return (double)blocks * 256 * iters * CH / (best * 1e-3);   // ops per second
}

int main() {
  int nsm = 0, clk = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int blocks = nsm * 8, iters = 20000;
  const char* names[4] = {"dfma", "dadd", "dmul", "ddiv_rn_seq"};
  for (int op = 0; op < 4; ++op) {
    float ms = 0;
    double r = op == 0 ? run<0>(blocks, iters, &ms) : op == 1 ? run<1>(blocks, iters, &ms)
             : op == 2 ? run<2>(blocks, iters, &ms) : run<3>(blocks, iters / 4, &ms);
    const double flops = (op == 0 ? 2.0 : 1.0) * r;
    printf("{\"op\": \"%s\", \"ops_per_s\": %.6e, \"tflops\": %.3f, \"per_sm_per_clk_at_max\": %.2f, "
           "\"ms\": %.3f, \"sms\": %d, \"max_clock_mhz\": %d}\n",
           names[op], r, flops / 1e12, r / nsm / (clk * 1e3), ms, nsm, clk / 1000);
  }
  return 0;
}
