// Scattered 128-byte rows per SM: LSU (cp.async 16 B x 8 threads per row /
// st.global.cg.v4) versus plain bulk copies (cp.async.bulk 128 B per row,
// mbarrier completion / bulk_group), the wave executor's per-line traffic
// shape (diagnostics, not part of the library). One CTA of 384 threads per
// SM moves `rows` random rows of a 205,888 x 128-float field per line,
// `lines` times; prints cycles per line.
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/bmb tools/bulk_microbench.cu
//   tools/bmb <mode 0..3> <rows per line>
//   modes: 0 LDGSTS gather, 1 bulk gather, 2 STG store, 3 bulk store
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int NT = 384, MAXR = 768, CELLS = 205888, SP = 128;

__device__ __forceinline__ uint32_t sa(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

__global__ void __launch_bounds__(NT, 1) bench(int mode, const float* __restrict__ f, float* __restrict__ g,
                                              const uint32_t* __restrict__ rows_all, int rows, int lines,
                                              unsigned long long* out, int split) {
    extern __shared__ __align__(128) float buf[];  // [MAXR][32]
    __shared__ __align__(8) uint64_t bar;
    const int t = threadIdx.x;
    if (t == 0)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&bar)), "r"(1) : "memory");
    __syncthreads();
    const uint32_t* rw = rows_all + size_t(blockIdx.x) * lines * rows;
    unsigned phase = 0;
    unsigned long long t0 = clock64();
    for (int l = 0; l < lines; ++l) {
        const uint32_t* r = rw + size_t(l) * rows;
        if (mode == 4) {  // half the rows by LDGSTS, half by bulk copies, at once
            const int h = rows / 2;
            if (t == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)),
                             "r"(unsigned((rows - h) * 128))
                             : "memory");
            __syncthreads();
            for (int row = h + t; row < rows; row += NT) {
                const float* src = f + size_t(r[row]) * SP;
                asm volatile(
                    "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], 128, [%2];" ::"r"(
                        sa(buf + row * 32)),
                    "l"(src), "r"(sa(&bar))
                    : "memory");
            }
            for (int i = t; i < h * 8; i += NT) {
                const int row = i / 8, q = i % 8;
                const float* src = f + size_t(r[row]) * SP + q * 4;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa(buf + row * 32 + q * 4)), "l"(src)
                             : "memory");
            }
            asm volatile("cp.async.commit_group; cp.async.wait_all;" ::: "memory");
            asm volatile(
                "{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(sa(&bar)),
                "r"(phase)
                : "memory");
            phase ^= 1;
            __syncthreads();
        } else if (mode == 0) {  // 8 threads x 16 B per row
            for (int i = t; i < rows * 8; i += NT) {
                const int row = i / 8, q = i % 8;
                const float* src = f + size_t(r[row]) * SP + q * 4;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa(buf + row * 32 + q * 4)), "l"(src)
                             : "memory");
            }
            asm volatile("cp.async.commit_group; cp.async.wait_all;" ::: "memory");
            __syncthreads();
        } else if (mode == 1) {  // one bulk copy of 128 B per row
            if (t == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)),
                             "r"(unsigned(rows * 128))
                             : "memory");
            __syncthreads();
            for (int row = t; row < rows; row += NT) {
                const float* src = f + size_t(r[row]) * SP;
                asm volatile(
                    "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], 128, [%2];" ::"r"(
                        sa(buf + row * 32)),
                    "l"(src), "r"(sa(&bar))
                    : "memory");
            }
            asm volatile(
                "{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(sa(&bar)),
                "r"(phase)
                : "memory");
            phase ^= 1;
            __syncthreads();
        } else if (mode == 2) {  // 8 threads x float4 per row
            for (int i = t; i < rows * 8; i += NT) {
                const int row = i / 8, q = i % 8;
                float* dst = g + size_t(r[row]) * SP + q * 4;
                const float4 v = *reinterpret_cast<const float4*>(buf + row * 32 + q * 4);
                asm volatile("st.global.cg.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(v.x), "f"(v.y), "f"(v.z),
                             "f"(v.w)
                             : "memory");
            }
            __syncthreads();
        } else if (mode == 5) {  // 4 threads x 32 B (st.global.v8) per row
            for (int i = t; i < rows * 4; i += NT) {
                const int row = i / 4, q = i % 4;
                float* dst = g + size_t(r[row]) * SP + q * 8;
                const float4 v0 = *reinterpret_cast<const float4*>(buf + row * 32 + q * 8);
                const float4 v1 = *reinterpret_cast<const float4*>(buf + row * 32 + q * 8 + 4);
                asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst), "f"(v0.x),
                             "f"(v0.y), "f"(v0.z), "f"(v0.w), "f"(v1.x), "f"(v1.y), "f"(v1.z), "f"(v1.w)
                             : "memory");
            }
            __syncthreads();
        } else if (mode == 6) {  // 4 threads x 32 B (ld.global.v8) per row into registers
            float acc = 0.f;
            for (int i = t; i < rows * 4; i += NT) {
                const int row = i / 4, q = i % 4;
                const float* src = f + size_t(r[row]) * SP + q * 8;
                float v[8];
                asm volatile("ld.global.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                             : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]),
                               "=f"(v[7])
                             : "l"(src));
                acc += v[0] + v[7];
            }
            if (acc == 12345.f)
                g[0] = acc;
            __syncthreads();
        } else if (mode == 7) {  // 8 threads x float4 ld.global into registers
            float acc = 0.f;
            for (int i = t; i < rows * 8; i += NT) {
                const int row = i / 8, q = i % 8;
                const float4 v = __ldcg(reinterpret_cast<const float4*>(f + size_t(r[row]) * SP + q * 4));
                acc += v.x + v.w;
            }
            if (acc == 12345.f)
                g[0] = acc;
            __syncthreads();
        } else if (mode == 8) {  // warps 0-5 gather this line's rows while warps 6-11 store another set
            if (t < NT / 2) {
                for (int i = t; i < rows * 8; i += NT / 2) {
                    const int row = i / 8, q = i % 8;
                    const float* src = f + size_t(r[row]) * SP + q * 4;
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa(buf + row * 32 + q * 4)),
                                 "l"(src)
                                 : "memory");
                }
                asm volatile("cp.async.commit_group; cp.async.wait_all;" ::: "memory");
            } else {
                const uint32_t* r2 = rw + size_t((l + 1) % lines) * rows;
                for (int i = t - NT / 2; i < rows * 8; i += NT / 2) {
                    const int row = i / 8, q = i % 8;
                    float* dst = g + size_t(r2[row]) * SP + q * 4;
                    const float4 v = *reinterpret_cast<const float4*>(buf + (MAXR / 2 + row % (MAXR / 2)) * 32 + q * 4);
                    asm volatile("st.global.cg.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(v.x), "f"(v.y),
                                 "f"(v.z), "f"(v.w)
                                 : "memory");
                }
            }
            __syncthreads();
        } else if (mode == 9) {  // every thread issues its gathers, then its stores, then waits
            const uint32_t* r2 = rw + size_t((l + 1) % lines) * rows;
            for (int i = t; i < rows * 8; i += NT) {
                const int row = i / 8, q = i % 8;
                const float* src = f + size_t(r[row]) * SP + q * 4;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa(buf + row * 32 + q * 4)), "l"(src)
                             : "memory");
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
            for (int i = t; i < rows * 8; i += NT) {
                const int row = i / 8, q = i % 8;
                float* dst = g + size_t(r2[row]) * SP + q * 4;
                const float4 v = *reinterpret_cast<const float4*>(buf + (MAXR / 2 + row % (MAXR / 2)) * 32 + q * 4);
                asm volatile("st.global.cg.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(v.x), "f"(v.y), "f"(v.z),
                             "f"(v.w)
                             : "memory");
            }
            asm volatile("cp.async.wait_all;" ::: "memory");
            __syncthreads();
        } else if (mode == 10 || mode == 11) {  // LSU gathers; stores: 10 all by TMA bulk, 11 the first `split` by TMA
            const uint32_t* r2 = rw + size_t((l + 1) % lines) * rows;
            const int k = mode == 10 ? rows : split;
            for (int row = t; row < k; row += NT) {
                float* dst = g + size_t(r2[row]) * SP;
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 128;" ::"l"(dst),
                             "r"(sa(buf + (MAXR / 2 + row % (MAXR / 2)) * 32))
                             : "memory");
            }
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            for (int i = t; i < rows * 8; i += NT) {
                const int row = i / 8, q = i % 8;
                const float* src = f + size_t(r[row]) * SP + q * 4;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa(buf + row * 32 + q * 4)), "l"(src)
                             : "memory");
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
            for (int i = t + k * 8; i < rows * 8; i += NT) {
                const int row = i / 8, q = i % 8;
                float* dst = g + size_t(r2[row]) * SP + q * 4;
                const float4 v = *reinterpret_cast<const float4*>(buf + (MAXR / 2 + row % (MAXR / 2)) * 32 + q * 4);
                asm volatile("st.global.cg.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(v.x), "f"(v.y), "f"(v.z),
                             "f"(v.w)
                             : "memory");
            }
            asm volatile("cp.async.wait_all;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            __syncthreads();
        } else if (mode == 3) {  // one bulk store of 128 B per row
            for (int row = t; row < rows; row += NT) {
                float* dst = g + size_t(r[row]) * SP;
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 128;" ::"l"(dst),
                             "r"(sa(buf + row * 32))
                             : "memory");
            }
            asm volatile("cp.async.bulk.commit_group; cp.async.bulk.wait_group.read 0;" ::: "memory");
            __syncthreads();
        }
    }
    if (mode == 3 || mode == 10 || mode == 11)
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __syncthreads();
    if (t == 0)
        out[blockIdx.x] = clock64() - t0;
}

int main(int argc, char** argv) {
    const int mode = argc > 1 ? atoi(argv[1]) : 0;
    const int rows = argc > 2 ? atoi(argv[2]) : 460;
    const int lines = 200;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    if (argc > 3)
        sms = atoi(argv[3]);
    const int split = argc > 5 ? atoi(argv[5]) : rows / 2;
    const bool same = argc > 4 && atoi(argv[4]) != 0;  // store into the gathered array (the wave's in-place field)
    float *f, *g;
    cudaMalloc(&f, sizeof(float) * size_t(CELLS) * SP);
    cudaMalloc(&g, sizeof(float) * size_t(CELLS) * SP);
    cudaMemset(f, 0, sizeof(float) * size_t(CELLS) * SP);
    if (same)
        g = f;
    std::vector<uint32_t> h(size_t(sms) * lines * rows);
    uint64_t s = 12345;
    for (auto& x : h) {
        s = s * 6364136223846793005ull + 1442695040888963407ull;
        x = uint32_t((s >> 33) % CELLS);
    }
    uint32_t* d;
    cudaMalloc(&d, sizeof(uint32_t) * h.size());
    cudaMemcpy(d, h.data(), sizeof(uint32_t) * h.size(), cudaMemcpyHostToDevice);
    unsigned long long* out;
    cudaMalloc(&out, sizeof(unsigned long long) * sms);
    const size_t smem = size_t(MAXR) * 32 * 4;
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    for (int rep = 0; rep < 2; ++rep)
        bench<<<sms, NT, smem>>>(mode, f, g, d, rows, lines, out, split);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(e));
        return 1;
    }
    std::vector<unsigned long long> ho(sms);
    cudaMemcpy(ho.data(), out, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost);
    double mean = 0;
    for (auto v : ho)
        mean += double(v);
    mean /= sms;
    const char* names[] = {"LDGSTS gather", "bulk gather", "STG store", "bulk store", "half+half",
                           "STG.256 store", "LDG.256 gather", "LDG.128 gather", "gather||store", "gather;store", "LSU gather+TMA store", "LSU gather+split store"};
    if (mode == 11)
        printf("[split %d] ", split);
    printf("%-14s rows/line %d: %.0f cycles per line (%.2f cycles per row) on %d SMs\n", names[mode], rows,
           mean / lines, mean / lines / rows, sms);
    return 0;
}
