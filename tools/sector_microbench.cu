// Random 4-byte gathers and read-modify-writes over a field larger than L2:
// the access pattern of the volume MART executor (C4: a 211 MB fp32 field,
// cells visited in ray order). Reports the DRAM-sector rate the memory system
// sustains for it (diagnostics, not part of the library).
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/smb tools/sector_microbench.cu
//   tools/smb <field MB> <mode 0 gather | 1 gather+store> <run length>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__global__ void k(const uint32_t* __restrict__ idx, uint64_t n, float* __restrict__ f, int mode, float* out) {
    float acc = 0.f;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t c = __ldcs(idx + i);
        const float v = __ldcg(f + c);
        acc += v;
        if (mode == 1)
            __stcg(f + c, v * 1.0001f);
    }
    if (acc == 1234.5f)
        out[0] = acc;
}

int main(int argc, char** argv) {
    const size_t mb = argc > 1 ? atoi(argv[1]) : 211;
    const int mode = argc > 2 ? atoi(argv[2]) : 0;
    const int run = argc > 3 ? atoi(argv[3]) : 1;  // consecutive cells per random start (a ray's sector runs)
    const size_t cells = mb * 1000000 / 4;
    const uint64_t n = uint64_t(1) << 28;
    std::vector<uint32_t> h(n);
    uint64_t s = 88172645463325252ull;
    for (uint64_t i = 0; i < n; i += run) {
        s ^= s << 13, s ^= s >> 7, s ^= s << 17;
        const uint32_t c = uint32_t(s % (cells - run));
        for (int r = 0; r < run && i + r < n; ++r)
            h[i + r] = c + r;
    }
    uint32_t* idx;
    float *f, *out;
    cudaMalloc(&idx, n * 4);
    cudaMalloc(&f, cells * 4);
    cudaMalloc(&out, 4);
    cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
    cudaMemset(f, 0, cells * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k<<<148 * 8, 256>>>(idx, n, f, mode, out);
    cudaEventRecord(a);
    for (int r = 0; r < 3; ++r)
        k<<<148 * 8, 256>>>(idx, n, f, mode, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    ms /= 3;
    const double acc = double(n) / (ms * 1e-3);
    printf("field %zu MB mode %d run %d: %.3f ms, %.2f G accesses/s, %.0f GB/s as 32-byte sectors, %.0f GB/s useful (4 B%s)\n",
           mb, mode, run, ms, acc / 1e9, acc * 32 / 1e9 * (mode ? 2 : 1), acc * 4 / 1e9 * (mode ? 2 : 1),
           mode ? " read + 4 B write" : "");
    return 0;
}
