// FP64 throughput microbenchmarks on the B200 (the FP64 roofline denominator
// MEASURED_PEAKS.json lacks): DFMA on the CUDA cores and DMMA.884
// (mma.sync.m8n8k4.f64) on the tensor cores, each alone, timed with CUDA
// events over a grid of 148 x 8 CTAs x 256 threads, best of 10.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
// prints one JSON line.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 1 << 14;
constexpr int kChains = 8;

__global__ void dfma_kernel(double* out, double a, double b) {
    double x[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-3 + c;
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) x[c] = fma(x[c], a, b);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += x[c];
    if (s == 1234.5) out[threadIdx.x] = s;  // never true: keeps the chains live
}

__global__ void dmma_kernel(double* out, double a, double b) {
    double d[kChains][2];
#pragma unroll
    for (int c = 0; c < kChains; ++c) d[c][0] = d[c][1] = threadIdx.x * 1e-3 + c;
    for (int it = 0; it < kIters / 4; ++it) {
#pragma unroll
        for (int c = 0; c < kChains; ++c)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
                         : "+d"(d[c][0]), "+d"(d[c][1])
                         : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += d[c][0] + d[c][1];
    if (s == 1234.5) out[threadIdx.x] = s;
}

// DFMA and DMMA chains interleaved in every warp: ~2x either alone if the
// tensor-core DMMA path and the FP64 FMA pipe issue independently
__global__ void mixed_kernel(double* out, double a, double b) {
    double x[kChains], d[kChains / 2][2];
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-3 + c;
#pragma unroll
    for (int c = 0; c < kChains / 2; ++c) d[c][0] = d[c][1] = threadIdx.x * 1e-3 + c;
    for (int it = 0; it < kIters / 4; ++it) {
#pragma unroll
        for (int c = 0; c < kChains / 2; ++c)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
                         : "+d"(d[c][0]), "+d"(d[c][1])
                         : "d"(a), "d"(b));
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < kChains; ++c) x[c] = fma(x[c], a, b);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += x[c];
#pragma unroll
    for (int c = 0; c < kChains / 2; ++c) s += d[c][0] + d[c][1];
    if (s == 1234.5) out[threadIdx.x] = s;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 8, threads = 256;
    double* out;
    cudaMalloc(&out, 1024 * sizeof(double));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double best[3] = {0, 0, 0};
    for (int k = 0; k < 3; ++k) {
        for (int rep = 0; rep < 12; ++rep) {
            cudaEventRecord(e0);
            if (k == 0) dfma_kernel<<<blocks, threads>>>(out, 0.999999, 1e-7);
            else if (k == 1) dmma_kernel<<<blocks, threads>>>(out, 0.999999, 1e-7);
            else mixed_kernel<<<blocks, threads>>>(out, 0.999999, 1e-7);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            double flops;
            if (k == 0) flops = 2.0 * kChains * kIters * double(blocks) * threads;
            else if (k == 1) flops = 512.0 * kChains * (kIters / 4) * double(blocks) * (threads / 32);
            else
                flops = (512.0 * (kChains / 2) * (threads / 32) + 2.0 * kChains * 4 * threads) * (kIters / 4) *
                        double(blocks);
            const double tf = flops / (ms * 1e-3) / 1e12;
            if (rep >= 2 && tf > best[k]) best[k] = tf;
        }
    }
    cudaError_t err = cudaGetLastError();
    printf("{\"dfma_tflops\": %.3f, \"dmma884_tflops\": %.3f, \"dfma_plus_dmma_interleaved_tflops\": %.3f, "
           "\"sms\": %d, \"error\": \"%s\"}\n",
           best[0], best[1], best[2], sms, cudaGetErrorString(err));
    return err == cudaSuccess ? 0 : 1;
}
