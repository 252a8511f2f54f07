// Scattered-row throughput: LSU (cp.async 16 B / st.global.cg float4) versus
// TMA tile::gather4 / tile::scatter4 (4 arbitrary rows of the [cells][Sp]
// field per instruction), for the MART line shape (diagnostics, not part of
// the library). Each group runs `lines` synthetic lines of n random cells:
// gather the line's P-wide rows into shared memory, sum them, scale, write
// them back. Cycles per line from clock64.
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -DTMB_P=8 -o tools/tmb8 tools/tma_microbench.cu
//   tools/tmb8 <groups_per_sm> <sms>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cfloat>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#ifndef TMB_P
#define TMB_P 8
#endif
constexpr int P = TMB_P, G = 256, NMAX = 640, ROWB = P * 4;

enum : int { kLoad = 1, kStore = 2, kTma = 4 };

__device__ __forceinline__ uint32_t sm_addr(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sm_addr(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sm_addr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
    asm volatile(
        "{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(sm_addr(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* m, uint64_t* bar, int col, int r0, int r1,
                                            int r2, int r3) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
        "%5, %6}], [%7];" ::"r"(sm_addr(dst)),
        "l"(m), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(sm_addr(bar))
        : "memory");
}
__device__ __forceinline__ void tma_scatter4(const CUtensorMap* m, const void* src, int col, int r0, int r1, int r2,
                                             int r3) {
    asm volatile(
        "cp.async.bulk.tensor.2d.global.shared::cta.tile::scatter4.bulk_group [%0, {%2, %3, %4, %5, %6}], [%1];" ::"l"(
            m),
        "r"(sm_addr(src)), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
        : "memory");
}

template <int FLAGS>
__global__ void __launch_bounds__(1024, 1)
    line_loop(const __grid_constant__ CUtensorMap tmap, float* field, const uint32_t* idx_all, int n, int lines,
              int Sp, unsigned long long* cyc, float* out) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int g = threadIdx.x / G, t = threadIdx.x % G, ng = blockDim.x / G;
    float* buf = reinterpret_cast<float*>(smem) + size_t(g) * NMAX * P;
    __shared__ uint64_t bars[4];
    __shared__ float red[4][G / 32][P];
    __shared__ float fac[4][P];
    __shared__ uint32_t sidx[4][NMAX];
    const int col = int(blockIdx.x % (Sp / P)) * P;
    const uint32_t* idx0 = idx_all + size_t(blockIdx.x * 4 + g) * lines * n;
    auto bar = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(G) : "memory"); };
    if (t == 0)
        mbar_init(&bars[g], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    const int n4 = (n + 3) & ~3;
    float acc = 0;
    const unsigned long long c0 = clock64();
    for (int j = 0; j < lines; ++j) {
        for (int s = t; s < n4; s += G)
            sidx[g][s] = __ldg(idx0 + size_t(j) * n + (s < n ? s : n - 1));
        bar();
        // ---- gather
        if (FLAGS & kLoad) {
            if (FLAGS & kTma) {
                if (t < 32) {
                    if (t == 0)
                        mbar_expect(&bars[g], unsigned(n4 * ROWB));
                    __syncwarp();
                    for (int q = t; q < n4 / 4; q += 32) {
                        const uint32_t* r = &sidx[g][4 * q];
                        tma_gather4(buf + 4 * q * P, &tmap, &bars[g], col, int(r[0]), int(r[1]), int(r[2]),
                                    int(r[3]));
                    }
                }
                mbar_wait(&bars[g], unsigned(j & 1));
            } else {
                for (int s = t; s < n4 * (P / 4); s += G) {
                    const int c = s / (P / 4), k = s % (P / 4);
                    const float* src = field + size_t(sidx[g][c]) * Sp + col + 4 * k;
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sm_addr(buf + 4 * s)), "l"(src)
                                 : "memory");
                }
                asm volatile("cp.async.commit_group; cp.async.wait_all;" ::: "memory");
                bar();
            }
        }
        // ---- sums (thread: one problem column p, a stride of cells)
        {
            const int p = t % P, c0_ = t / P;
            float s = 0;
            for (int c = c0_; c < n; c += G / P)
                s += buf[c * P + p];
            for (int o = P; o < 32; o <<= 1)
                s += __shfl_xor_sync(~0u, s, o);
            if ((t & 31) < P)
                red[g][t >> 5][p] = s;
        }
        bar();
        if (t < P) {
            float pb = 0;
            for (int w = 0; w < G / 32; ++w)
                pb += red[g][w][t];
            fac[g][t] = 1.0f - 0.05f * (1.0f - 100.0f / fmaxf(pb, 1e-12f));
        }
        bar();
        // ---- scale in place
        for (int s = t; s < n4 * P; s += G)
            buf[s] = fmaxf(buf[s] * fac[g][s % P], FLT_MIN);
        // ---- scatter
        if (FLAGS & kStore) {
            if (FLAGS & kTma) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                bar();
                if (t < 32) {
                    for (int q = t; q < n4 / 4; q += 32) {
                        const uint32_t* r = &sidx[g][4 * q];
                        tma_scatter4(&tmap, buf + 4 * q * P, col, int(r[0]), int(r[1]), int(r[2]), int(r[3]));
                    }
                    asm volatile("cp.async.bulk.commit_group; cp.async.bulk.wait_group.read 0;" ::: "memory");
                }
            } else {
                for (int s = t; s < n4 * (P / 4); s += G) {
                    const int c = s / (P / 4), k = s % (P / 4);
                    if (c < n)
                        __stcg(reinterpret_cast<float4*>(field + size_t(sidx[g][c]) * Sp + col) + k,
                               reinterpret_cast<const float4*>(buf)[s]);
                }
            }
        }
        acc += buf[t];
        bar();
    }
    if (t == 0) {
        cyc[blockIdx.x * 4 + g] = clock64() - c0;
    }
    if (acc == -1.f)
        out[0] = acc;
    (void)ng;
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}

template <int FLAGS>
static double run(const CUtensorMap& m, float* field, const uint32_t* idx, int n, int lines, int Sp, int groups,
                  int sms, unsigned long long* d_cyc, float* out) {
    const size_t smem = size_t(groups) * NMAX * P * sizeof(float);
    cudaFuncSetAttribute(line_loop<FLAGS>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    line_loop<FLAGS><<<sms, G * groups, smem>>>(m, field, idx, n, lines, Sp, d_cyc, out);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        std::printf("error: %s\n", cudaGetErrorString(e));
        std::exit(1);
    }
    std::vector<unsigned long long> c(size_t(sms) * 4);
    cudaMemcpy(c.data(), d_cyc, c.size() * 8, cudaMemcpyDeviceToHost);
    double s = 0;
    int k = 0;
    for (int b = 0; b < sms; ++b)
        for (int g = 0; g < groups; ++g, ++k)
            s += double(c[size_t(b) * 4 + g]);
    return s / k / lines;
}

// correctness: one group gathers + scatters (factor) a known line; check the field on the host
static bool check(const CUtensorMap& m, float* field, size_t cells, int Sp, unsigned long long* cyc, float* out) {
    std::vector<float> h(cells * Sp);
    for (size_t i = 0; i < h.size(); ++i)
        h[i] = float((i * 2654435761u) % 1000) / 250.0f + 0.5f;
    cudaMemcpy(field, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    const int n = 37;
    std::vector<uint32_t> id(size_t(4) * n);
    for (int i = 0; i < n; ++i)
        id[i] = uint32_t((i * 7919u + 11) % cells);
    uint32_t* d;
    cudaMalloc(&d, id.size() * 4);
    cudaMemcpy(d, id.data(), id.size() * 4, cudaMemcpyHostToDevice);
    auto ref = h;
    {
        const int col = 0;
        for (int p = 0; p < P; ++p) {
            float pb = 0;
            for (int i = 0; i < n; ++i)
                pb += ref[size_t(id[i]) * Sp + col + p];
            const float f = 1.0f - 0.05f * (1.0f - 100.0f / pb);
            for (int i = 0; i < n; ++i)
                ref[size_t(id[i]) * Sp + col + p] = fmaxf(ref[size_t(id[i]) * Sp + col + p] * f, FLT_MIN);
        }
    }
    const size_t smem = NMAX * P * sizeof(float);
    cudaFuncSetAttribute(line_loop<kLoad | kStore | kTma>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    line_loop<kLoad | kStore | kTma><<<1, G, smem>>>(m, field, d, n, 1, Sp, cyc, out);
    cudaDeviceSynchronize();
    std::vector<float> got(h.size());
    cudaMemcpy(got.data(), field, got.size() * 4, cudaMemcpyDeviceToHost);
    double md = 0;
    size_t bad = 0;
    for (size_t i = 0; i < h.size(); ++i) {
        const double dd = std::abs(double(got[i]) - double(ref[i])) / std::abs(double(ref[i]));
        if (dd > 1e-5)
            ++bad;
        md = dd > md ? dd : md;
    }
    std::printf("check: %zu mismatches, max rel %.3g (%s)\n", bad, md, cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
    return bad == 0;
}

int main(int argc, char** argv) {
    const int groups = argc > 1 ? std::atoi(argv[1]) : 1;
    const int sms = argc > 2 ? std::atoi(argv[2]) : 148;
    const int boxrows = argc > 3 ? std::atoi(argv[3]) : 1;
    const int n = 574, lines = 256, Sp = 128;
    const size_t cells = 205888;
    float *field, *out;
    uint32_t* idx;
    unsigned long long* cyc;
    cudaMalloc(&field, cells * Sp * sizeof(float));
    cudaMalloc(&out, 16);
    cudaMalloc(&idx, size_t(sms) * 4 * lines * n * sizeof(uint32_t));
    cudaMalloc(&cyc, size_t(sms) * 4 * 8);
    CUtensorMap m;
    const cuuint64_t dims[2] = {cuuint64_t(Sp), cuuint64_t(cells)};
    const cuuint64_t strides[1] = {cuuint64_t(Sp) * 4};
    const cuuint32_t box[2] = {cuuint32_t(P), cuuint32_t(boxrows)};
    const cuuint32_t es[2] = {1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, field, dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    std::printf("encode(box %d x %d) = %d\n", P, boxrows, int(r));
    if (!check(m, field, cells, Sp, cyc, out))
        return 1;
    std::vector<float> ones(cells * Sp, 1.0f);
    cudaMemcpy(field, ones.data(), ones.size() * 4, cudaMemcpyHostToDevice);
    std::vector<uint32_t> h(size_t(sms) * 4 * lines * n);
    uint64_t st = 12345;
    for (auto& v : h) {
        st = st * 6364136223846793005ull + 1442695040888963407ull;
        v = uint32_t((st >> 33) % cells);
    }
    cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    std::printf("P=%d groups/SM=%d SMs=%d n=%d: cycles per line\n", P, groups, sms, n);
    for (int rep = 0; rep < 2; ++rep) {
        std::printf("  lsu  load+store %.0f  load %.0f  store %.0f  none %.0f\n",
                    run<kLoad | kStore>(m, field, idx, n, lines, Sp, groups, sms, cyc, out),
                    run<kLoad>(m, field, idx, n, lines, Sp, groups, sms, cyc, out),
                    run<kStore>(m, field, idx, n, lines, Sp, groups, sms, cyc, out),
                    run<0>(m, field, idx, n, lines, Sp, groups, sms, cyc, out));
        std::printf("  tma  load+store %.0f  load %.0f  store %.0f\n",
                    run<kLoad | kStore | kTma>(m, field, idx, n, lines, Sp, groups, sms, cyc, out),
                    run<kLoad | kTma>(m, field, idx, n, lines, Sp, groups, sms, cyc, out),
                    run<kStore | kTma>(m, field, idx, n, lines, Sp, groups, sms, cyc, out));
    }
    std::printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
