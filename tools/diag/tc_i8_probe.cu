// Probe: tcgen05.mma.kind::i8 (u8 x u8 -> s32) with K-major SWIZZLE_NONE
// shared-memory operands, accumulator in TMEM, read back with
// tcgen05.ld.32x32b. Checks D = A * B^T against the host for a few
// (LBO, SBO) descriptor conventions and N sizes. Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/tcp tools/diag/tc_i8_probe.cu && /tmp/tcp
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess) {                                                       \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            exit(1);                                                                   \
        }                                                                              \
    } while (0)

constexpr int M = 128, KB = 64;

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= uint64_t((saddr >> 4) & 0x3FFF);
    d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
    d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
    d |= uint64_t(1) << 46;  // version (sm_100)
    // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
    return d;
}

__global__ void probe(const uint8_t* A, const uint8_t* B, int32_t* D, int N, int variant) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* sa = sm;                 // M x KB
    uint8_t* sb = sm + M * KB;        // N x KB
    __shared__ uint64_t bar;
    __shared__ uint32_t taddr_s;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    // core-matrix layout: (row, kc) at (row/8)*SBO + kc*LBO + (row%8)*16, LBO=128, SBO=KB/16*128
    const uint32_t LBO = 128, SBO = (KB / 16) * 128;
    for (int e = t; e < M * (KB / 16); e += blockDim.x) {
        int row = e / (KB / 16), kc = e % (KB / 16);
        const uint4 v = *reinterpret_cast<const uint4*>(A + row * KB + kc * 16);
        *reinterpret_cast<uint4*>(sa + (row / 8) * SBO + kc * LBO + (row % 8) * 16) = v;
    }
    for (int e = t; e < N * (KB / 16); e += blockDim.x) {
        int row = e / (KB / 16), kc = e % (KB / 16);
        const uint4 v = *reinterpret_cast<const uint4*>(B + row * KB + kc * 16);
        *reinterpret_cast<uint4*>(sb + (row / 8) * SBO + kc * LBO + (row % 8) * 16) = v;
    }
    if (warp == 0) {
        const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(&taddr_s));
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(dst));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (t == 0) {
        const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(&bar));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(b));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = taddr_s;
    if (t == 0) {
        uint32_t idesc = 0;
        idesc |= 2u << 4;                     // D = s32
        idesc |= 0u << 7;                     // A u8
        idesc |= 0u << 10;                    // B u8
        idesc |= uint32_t(N >> 3) << 17;      // N
        idesc |= uint32_t(M >> 4) << 24;      // M
        const uint32_t a0 = static_cast<uint32_t>(__cvta_generic_to_shared(sa));
        const uint32_t b0 = static_cast<uint32_t>(__cvta_generic_to_shared(sb));
        uint32_t lbo = LBO, sbo = SBO;
        if (variant == 1) { lbo = SBO; sbo = LBO; }
        for (int k = 0; k < KB / 32; ++k) {
            const uint64_t ad = sdesc(a0 + k * 2 * LBO, lbo, sbo);
            const uint64_t bd = sdesc(b0 + k * 2 * LBO, lbo, sbo);
            const uint32_t acc = k > 0;
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
        }
        const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(&bar));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(b)
                     : "memory");
    }
    {
        const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(&bar));
        asm volatile(
            "{\n.reg .pred P1;\nWAIT_%=:\n"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
            "@!P1 bra WAIT_%=;\n}\n" ::"r"(b)
            : "memory");
    }
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const int row = 32 * (warp & 3) + lane;
    for (int c = 0; c < N; c += 8) {
        uint32_t r[8];
        const uint32_t ta = tmem + (uint32_t(32 * (warp & 3)) << 16) + uint32_t(c);
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                       "=r"(r[7])
                     : "r"(ta));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        if (warp < 4)
            for (int j = 0; j < 8; ++j) D[row * N + c + j] = int32_t(r[j]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" ::"r"(tmem));
}

int main() {
    int bad_total = 0;
    for (int N : {176, 240, 32}) {
        std::vector<uint8_t> A(M * KB), B(N * KB);
        srand(7 + N);
        for (auto& x : A) x = uint8_t(rand());
        for (auto& x : B) x = uint8_t(rand());
        std::vector<int32_t> ref(M * N);
        for (int i = 0; i < M; ++i)
            for (int j = 0; j < N; ++j) {
                int32_t s = 0;
                for (int k = 0; k < KB; ++k) s += int32_t(A[i * KB + k]) * int32_t(B[j * KB + k]);
                ref[i * N + j] = s;
            }
        uint8_t *dA, *dB;
        int32_t* dD;
        CK(cudaMalloc(&dA, A.size()));
        CK(cudaMalloc(&dB, B.size()));
        CK(cudaMalloc(&dD, ref.size() * 4));
        CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
        const size_t smem = size_t(M + N) * KB + 1024;
        CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        for (int variant = 0; variant < 2; ++variant) {
            CK(cudaMemset(dD, 0xFF, ref.size() * 4));
            probe<<<1, 256, smem>>>(dA, dB, dD, N, variant);
            CK(cudaGetLastError());
            CK(cudaDeviceSynchronize());
            std::vector<int32_t> got(ref.size());
            CK(cudaMemcpy(got.data(), dD, got.size() * 4, cudaMemcpyDeviceToHost));
            int bad = 0;
            for (size_t i = 0; i < got.size(); ++i) bad += got[i] != ref[i];
            printf("N=%d variant=%d (%s): mismatches %d / %zu  (D[0]=%d ref %d, D[1]=%d ref %d, D[N]=%d ref %d)\n",
                   N, variant, variant ? "LBO=SBO-stride swapped" : "LBO=K-core stride", bad, got.size(), got[0],
                   ref[0], got[1], ref[1], got[N], ref[N]);
            if (variant == 0) bad_total += bad;
        }
        cudaFree(dA);
        cudaFree(dB);
        cudaFree(dD);
    }
    printf(bad_total ? "PROBE FAIL\n" : "PROBE OK\n");
    return 0;
}
