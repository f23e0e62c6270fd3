// Can a small low-priority kernel B run beside a persistent kernel A that holds one CTA of
// W warps x 128 registers and 174 KB of shared memory on every SM?  (The Γ pipeline's side
// stream question: DESIGN.md §4, "operand exposure".)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o coresidency tools/coresidency.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

template <int NA>
__global__ void __launch_bounds__(512, 1) spin_a(long long cycles, double* sink) {
    extern __shared__ double sm[];
    double acc[NA];  // keep registers live (the launch bound allows 128)
#pragma unroll
    for (int i = 0; i < NA; ++i) acc[i] = threadIdx.x * 0.5 + i;
    const long long t0 = clock64();
    while (clock64() - t0 < cycles) {
#pragma unroll
        for (int i = 0; i < NA; ++i) acc[i] = acc[i] * 1.0000001 + 0.5;
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < NA; ++i) s += acc[i];
    if (s == 123.456) sink[0] = s + sm[threadIdx.x];
}

__global__ void small_b(double* out, int n, int iters) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double v = i;
        for (int k = 0; k < iters; ++k) v = v * 1.0000001 + 1.0;
        out[i] = v;
    }
}

int main(int argc, char** argv) {
    const int warpsA = argc > 1 ? atoi(argv[1]) : 13;
    const int threadsB = argc > 2 ? atoi(argv[2]) : 128;
    const int order = argc > 3 ? atoi(argv[3]) : 0;  // 0: A first, 1: B first
    const int maxregA = argc > 4 ? atoi(argv[4]) : 128;
    int lo, hi;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    cudaStream_t sa, sb;
    cudaStreamCreateWithPriority(&sa, cudaStreamNonBlocking, hi);
    cudaStreamCreateWithPriority(&sb, cudaStreamNonBlocking, lo);
    double *sink, *out;
    const int n = 1 << 22;
    cudaMalloc(&sink, 8);
    cudaMalloc(&out, n * 8);
    const size_t shm = 178176;
    cudaFuncSetAttribute(spin_a<57>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, spin_a<57>);
    cudaEvent_t a0, a1, b0, b1;
    for (cudaEvent_t* e : {&a0, &a1, &b0, &b1}) cudaEventCreate(e);
    const long long cycles = 10LL * 1965000;  // ~10 ms
    for (int rep = 0; rep < 3; ++rep) {
        cudaDeviceSynchronize();
        if (order == 1) {
            cudaEventRecord(b0, sb);
            small_b<<<4096, threadsB, 0, sb>>>(out, n, 64);
            cudaEventRecord(b1, sb);
        }
        cudaEventRecord(a0, sa);
        spin_a<57><<<148, warpsA * 32, shm, sa>>>(cycles, sink);
        cudaEventRecord(a1, sa);
        if (order == 0) {
            cudaEventRecord(b0, sb);
            small_b<<<4096, threadsB, 0, sb>>>(out, n, 64);
            cudaEventRecord(b1, sb);
        }
        cudaDeviceSynchronize();
        float ta, tb, gap;
        cudaEventElapsedTime(&ta, a0, a1);
        cudaEventElapsedTime(&tb, b0, b1);
        cudaEventElapsedTime(&gap, a0, b1);
        printf("A %d warps (%d regs/thread compiled, %s first), B %d threads: A %.3f ms, B %.3f ms, "
               "B ends %.3f ms after A starts\n", warpsA, fa.numRegs, order ? "B" : "A", threadsB,
               ta, tb, gap);
    }
    (void)maxregA;
    return 0;
}
