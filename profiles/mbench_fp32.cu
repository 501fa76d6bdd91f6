// FP32 issue-rate microbenchmark on the box's GPU: scalar FFMA (register and immediate
// operand forms) vs packed FFMA2 / FADD2 / FMUL2 (sm_100a f32x2).  Each thread runs 8
// independent dependency chains (enough ILP at full occupancy); results in lane-FLOP/s
// (FMA = 2 flops, add / mul = 1) and warp-instructions per clock per SM.
// Build + run: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb profiles/mbench_fp32.cu && ./mb
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096, kChains = 8;

__global__ void ffma_reg(float* out, float a, float b) {
  float x[kChains];
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-3f + c;
  float y = b * (1.0f + threadIdx.x * 1e-9f);  // register operand, not an immediate
  for (int i = 0; i < kIters; ++i)
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = fmaf(x[c], a, y);
  float s = 0;
  for (int c = 0; c < kChains; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void ffma_imm(float* out, float a) {
  float x[kChains];
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-3f + c;
  for (int i = 0; i < kIters; ++i)
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = fmaf(x[c], 0.999f, 1e-3f);
  float s = 0;
  for (int c = 0; c < kChains; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + a;
}
__global__ void ffma2_reg(float* out, float a, float b) {
  float2 x[kChains];
  for (int c = 0; c < kChains; ++c) x[c] = make_float2(threadIdx.x * 1e-3f + c, c);
  const float2 av = make_float2(a, a * 0.5f), yv = make_float2(b, b * (1.0f + threadIdx.x * 1e-9f));
  for (int i = 0; i < kIters; ++i)
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = __ffma2_rn(x[c], av, yv);
  float s = 0;
  for (int c = 0; c < kChains; ++c) s += x[c].x + x[c].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void fadd2_reg(float* out, float a) {
  float2 x[kChains];
  for (int c = 0; c < kChains; ++c) x[c] = make_float2(threadIdx.x * 1e-3f + c, c);
  const float2 av = make_float2(a, a * (1.0f + threadIdx.x * 1e-9f));
  for (int i = 0; i < kIters; ++i)
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = __fadd2_rn(x[c], av);
  float s = 0;
  for (int c = 0; c < kChains; ++c) s += x[c].x + x[c].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void fmul2_reg(float* out, float a) {
  float2 x[kChains];
  for (int c = 0; c < kChains; ++c) x[c] = make_float2(threadIdx.x * 1e-3f + c, c + 1);
  const float2 av = make_float2(a, a * (1.0f + threadIdx.x * 1e-9f));
  for (int i = 0; i < kIters; ++i)
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = __fmul2_rn(x[c], av);
  float s = 0;
  for (int c = 0; c < kChains; ++c) s += x[c].x + x[c].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const int sms = p.multiProcessorCount, threads = 256, blocks = sms * 8;
  float* out;
  cudaMalloc(&out, sizeof(float) * blocks * threads);
  cudaEvent_t t0, t1;
  cudaEventCreate(&t0);
  cudaEventCreate(&t1);
  const double lanes = (double)blocks * threads, ops = lanes * kIters * kChains;
  auto run = [&](const char* name, auto launch, double flop_per_op, double lanes_per_inst) {
    launch();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(t0);
      launch();
      cudaEventRecord(t1);
      cudaEventSynchronize(t1);
      float ms;
      cudaEventElapsedTime(&ms, t0, t1);
      if (ms < best) best = ms;
    }
    const double s = best * 1e-3;
    const double warp_inst = ops / 32.0 / lanes_per_inst;  // instructions of the chain body
    const double clk = clk_khz * 1e3;
    printf("%-10s %8.3f ms  %7.2f TFLOP/s  %5.2f warp-inst/clk/SM\n", name, best, ops * flop_per_op / s * 1e-12,
           warp_inst / s / clk / sms);
  };
  run("ffma_reg", [&] { ffma_reg<<<blocks, threads>>>(out, 0.999f, 1e-3f); }, 2.0, 1.0);
  run("ffma_imm", [&] { ffma_imm<<<blocks, threads>>>(out, 0.f); }, 2.0, 1.0);
  run("ffma2_reg", [&] { ffma2_reg<<<blocks, threads>>>(out, 0.999f, 1e-3f); }, 4.0, 1.0);
  run("fadd2_reg", [&] { fadd2_reg<<<blocks, threads>>>(out, 1e-3f); }, 2.0, 1.0);
  run("fmul2_reg", [&] { fmul2_reg<<<blocks, threads>>>(out, 0.9999f); }, 2.0, 1.0);
  printf("SMs %d, max SM clock %.0f MHz (attribute), nominal FP32 peak %.1f TFLOP/s\n", sms, clk_khz / 1e3,
         sms * 128.0 * 2 * clk_khz * 1e3 * 1e-12);
  return 0;
}
