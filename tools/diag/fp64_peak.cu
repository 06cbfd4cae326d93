// FP64 pipe throughput probe: independent DFMA / DADD chains per thread at
// full occupancy; prints DP ops per clock per SM (B200 nominal: 64).
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void __launch_bounds__(256) k(double* out, double a, double b, int iters) {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) x[i] = __fma_rn(x[i], a, b);
            else if (OP == 1) x[i] = __dadd_rn(x[i], b);
            else x[i] = __dmul_rn(x[i], a);
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.678) out[0] = s;
}
int main() {
    double* out;
    cudaMalloc(&out, 8);
    int sms, clk;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int iters = 4096, blocks = sms * 8;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char* names[3] = {"DFMA", "DADD", "DMUL"};
    for (int op = 0; op < 3; ++op) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            if (op == 0) k<0><<<blocks, 256>>>(out, 1.0000001, 1e-9, iters);
            if (op == 1) k<1><<<blocks, 256>>>(out, 1.0000001, 1e-9, iters);
            if (op == 2) k<2><<<blocks, 256>>>(out, 1.0000001, 1e-9, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            double ops = double(blocks) * 256 * iters * 8;
            if (rep) printf("%s: %.2f Tops/s, %.1f ops/clk/SM at %d MHz nominal\n", names[op], ops / ms / 1e9,
                            ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
        }
    }
    return 0;
}
