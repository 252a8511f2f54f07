// Intrinsic per-line cost of the pipelined MART line loop (diagnostics, not
// part of the library): one or more independent 256-thread groups per SM,
// each running `lines` synthetic lines of n random cells of an [cells][Sp]
// fp32 field, P = 8 problems per task. Variants drop one ingredient at a time.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/lmb tools/line_microbench.cu
//   /tmp/lmb <groups_per_sm> <sms>
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#ifndef LMB_P
#define LMB_P 8
#endif
// P = 8: 256-thread groups (up to 4 per SM); P = 32: one 1024-thread group
constexpr int P = LMB_P, G = P == 8 ? 256 : 1024, TPC = P / 4, NCLV = G / TPC, KV = 6, MAXC = KV * NCLV;
constexpr int NG = 1024 / G;

enum : int { kGather = 1, kStore = 2, kF64 = 4, kF32Part = 8, kSmemIdx = 16, kRegLoad = 32 };

__device__ __forceinline__ void cp_async16_if(bool p, void* s, const void* g) {
    const unsigned d = unsigned(__cvta_generic_to_shared(s));
    asm volatile("{ .reg .pred q; setp.ne.b32 q, %2, 0; @q cp.async.cg.shared.global [%0], [%1], 16; }" ::"r"(d),
                 "l"(g), "r"(int(p))
                 : "memory");
}

template <int FLAGS>
__global__ void __launch_bounds__(1024, 1)
    line_loop(float* field, const uint32_t* idx_all, int n, int lines, int Sp, unsigned long long* cyc) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int g = threadIdx.x / G, t = threadIdx.x % G;
    float4* buf = reinterpret_cast<float4*>(smem) + size_t(g) * MAXC * TPC;
    __shared__ double red[NG][G / 32][P];
    __shared__ float2 fac[NG][P];
    const int q = t % TPC, cl = t / TPC;
    const uint32_t Sp4 = Sp / 4, col4 = (blockIdx.x % (Sp / P)) * (P / 4) + q;
    float4* f4 = reinterpret_cast<float4*>(field);
    const uint32_t* idx0 = idx_all + size_t(blockIdx.x * 4 + g) * lines * n;
    auto bar = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(G) : "memory"); };
    __shared__ uint32_t sidx[NG][2][MAXC];  // kSmemIdx: the line's indices staged (double-buffered)
    auto stage = [&](int j) {
        const uint32_t* idx = idx0 + size_t(j) * n;
        for (int s = t; s < n; s += G)
            sidx[g][j & 1][s] = __ldg(idx + s);
    };
    auto index = [&](int j, int s) -> uint32_t {
        if (FLAGS & kSmemIdx)
            return sidx[g][j & 1][s];
        return __ldg(idx0 + size_t(j) * n + s);
    };
    auto issue = [&](int j) {
        if (FLAGS & kRegLoad)
            return;
#pragma unroll
        for (int i = 0; i < KV; ++i) {
            const int s = cl + i * NCLV;
            const uint32_t e = index(j, s < n ? s : 0);
            if (FLAGS & kGather)
                cp_async16_if(s < n, buf + s * TPC + q, f4 + e * Sp4 + col4);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    if (FLAGS & kSmemIdx) {
        stage(0);
        bar();
    }
    issue(0);
    const unsigned long long c0 = clock64();
    // per-phase cycles of thread 0: [0] wait + sums [1] next issue [2] reduce + barrier
    // [3] factor + barrier [4] scale + stores [5] end barrier
    unsigned long long ph[6] = {0, 0, 0, 0, 0, 0};
    unsigned long long tk = clock64();
    auto stamp = [&](int k) {
        const unsigned long long now = clock64();
        ph[k] += now - tk;
        tk = now;
    };
    for (int j = 0; j < lines; ++j) {
        asm volatile("cp.async.wait_all;" ::: "memory");
        float4 x[KV];
        double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
        if (FLAGS & kRegLoad) {
            float a0 = 0, a1 = 0, a2 = 0, a3 = 0;
#pragma unroll
            for (int i = 0; i < KV; ++i) {
                const int s = cl + i * NCLV;
                x[i] = s < n ? __ldcg(f4 + index(j, s) * Sp4 + col4) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int i = 0; i < KV; ++i) {
                a0 += x[i].x;
                a1 += x[i].y;
                a2 += x[i].z;
                a3 += x[i].w;
            }
            s0 = a0, s1 = a1, s2 = a2, s3 = a3;
        } else if (FLAGS & kF32Part) {
            float a0 = 0, a1 = 0, a2 = 0, a3 = 0;
#pragma unroll
            for (int i = 0; i < KV; ++i) {
                const int s = cl + i * NCLV;
                x[i] = s < n ? buf[s * TPC + q] : make_float4(0.f, 0.f, 0.f, 0.f);
                a0 += x[i].x;
                a1 += x[i].y;
                a2 += x[i].z;
                a3 += x[i].w;
            }
            s0 = a0, s1 = a1, s2 = a2, s3 = a3;
        } else {
#pragma unroll
        for (int i = 0; i < KV; ++i) {
            const int s = cl + i * NCLV;
            x[i] = s < n ? buf[s * TPC + q] : make_float4(0.f, 0.f, 0.f, 0.f);
            s0 += double(x[i].x);
            s1 += double(x[i].y);
            s2 += double(x[i].z);
            s3 += double(x[i].w);
        }
        }
        asm volatile("" ::"d"(s0), "d"(s1), "d"(s2), "d"(s3));
        stamp(0);
        if (j + 1 < lines) {
            if (FLAGS & kSmemIdx)
                stage(j + 1);  // issued after the reduction barrier (other threads' entries)
            else
                issue(j + 1);
        }
        stamp(1);
#pragma unroll
        for (int o = TPC; o < 32; o <<= 1) {
            s0 += __shfl_xor_sync(~0u, s0, o);
            s1 += __shfl_xor_sync(~0u, s1, o);
            s2 += __shfl_xor_sync(~0u, s2, o);
            s3 += __shfl_xor_sync(~0u, s3, o);
        }
        const int lane = t & 31, warp = t >> 5;
        if (lane < TPC) {
            red[g][warp][q * 4 + 0] = s0;
            red[g][warp][q * 4 + 1] = s1;
            red[g][warp][q * 4 + 2] = s2;
            red[g][warp][q * 4 + 3] = s3;
        }
        bar();
        if ((FLAGS & kSmemIdx) && j + 1 < lines)
            issue(j + 1);
        stamp(2);
        if (t < P) {
            double pb = 0;
#pragma unroll
            for (int w = 0; w < G / 32; ++w)
                pb += red[g][w][t];
            double f;
            if (FLAGS & kF64)
                f = 1.0 - 0.05 * (1.0 - 100.0 / (pb > 1e-12 ? pb : 1e-12));
            else
                f = 1.0 - 0.05 * (1.0 - __fdividef(100.f, float(pb)));
            fac[g][t] = make_float2(float(f), FLT_MIN);
        }
        bar();
        stamp(3);
        const float4 u = reinterpret_cast<const float4*>(fac[g])[2 * q];
        const float4 w = reinterpret_cast<const float4*>(fac[g])[2 * q + 1];
#pragma unroll
        for (int i = 0; i < KV; ++i) {
            const int s = cl + i * NCLV;
            if (s < n) {
                const float4 r = make_float4(fmaxf(x[i].x * u.x, u.y), fmaxf(x[i].y * u.z, u.w),
                                             fmaxf(x[i].z * w.x, w.y), fmaxf(x[i].w * w.z, w.w));
                if (FLAGS & kStore)
                    __stcg(f4 + index(j, s) * Sp4 + col4, r);
                else
                    buf[s * TPC + q] = r;
            }
        }
        stamp(4);
        bar();
        stamp(5);
    }
    if (t == 0) {
        cyc[blockIdx.x * 4 + g] = clock64() - c0;
        if (blockIdx.x == 0 && g == 0)
            for (int k = 0; k < 6; ++k)
                cyc[gridDim.x * 4 + k] = ph[k] / lines;
    }
}

template <int FLAGS>
static double run(float* field, const uint32_t* idx, int n, int lines, int Sp, int groups, int sms,
                  unsigned long long* d_cyc) {
    const size_t smem = size_t(NG) * MAXC * TPC * sizeof(float4);
    cudaFuncSetAttribute(line_loop<FLAGS>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    line_loop<FLAGS><<<sms, G * groups, smem>>>(field, idx, n, lines, Sp, d_cyc);
    cudaDeviceSynchronize();
    std::vector<unsigned long long> c(size_t(sms) * 4 + 6);
    cudaMemcpy(c.data(), d_cyc, c.size() * 8, cudaMemcpyDeviceToHost);
    std::printf("    phases (block 0): wait+sum %llu issue %llu reduce %llu factor %llu store %llu endbar %llu\n",
                c[size_t(sms) * 4 + 0], c[size_t(sms) * 4 + 1], c[size_t(sms) * 4 + 2], c[size_t(sms) * 4 + 3],
                c[size_t(sms) * 4 + 4], c[size_t(sms) * 4 + 5]);
    double s = 0;
    int k = 0;
    for (int b = 0; b < sms; ++b)
        for (int g = 0; g < groups; ++g, ++k)
            s += double(c[size_t(b) * 4 + g]);
    return s / k / lines;
}

int main(int argc, char** argv) {
    const int groups = argc > 1 ? std::atoi(argv[1]) : 1;
    const int sms = argc > 2 ? std::atoi(argv[2]) : 148;
    const int n = 574, lines = 256, Sp = 128;
    const size_t cells = 205888;
    float* field;
    uint32_t* idx;
    unsigned long long* cyc;
    cudaMalloc(&field, cells * Sp * sizeof(float));
    cudaMalloc(&idx, size_t(sms) * 4 * lines * n * sizeof(uint32_t));
    cudaMalloc(&cyc, (size_t(sms) * 4 + 6) * 8);
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
        std::printf("  full (gather+store+f64)  %.0f\n", run<kGather | kStore | kF64>(field, idx, n, lines, Sp, groups, sms, cyc));
        std::printf("  no gather                %.0f\n", run<kStore | kF64>(field, idx, n, lines, Sp, groups, sms, cyc));
        std::printf("  no store                 %.0f\n", run<kGather | kF64>(field, idx, n, lines, Sp, groups, sms, cyc));
        std::printf("  no gather, no store      %.0f\n", run<kF64>(field, idx, n, lines, Sp, groups, sms, cyc));
        std::printf("  f32 factor (full mem)    %.0f\n", run<kGather | kStore>(field, idx, n, lines, Sp, groups, sms, cyc));
        std::printf("  f32 partials (full mem)  %.0f\n", run<kGather | kStore | kF64 | kF32Part>(field, idx, n, lines, Sp, groups, sms, cyc));
        std::printf("  f32 partials, no mem     %.0f\n", run<kF64 | kF32Part>(field, idx, n, lines, Sp, groups, sms, cyc));
        std::printf("  smem idx, f32 part, full %.0f\n", run<kGather | kStore | kF64 | kF32Part | kSmemIdx>(field, idx, n, lines, Sp, groups, sms, cyc));
        std::printf("  smem idx, reg loads, full %.0f\n", run<kGather | kStore | kF64 | kF32Part | kSmemIdx | kRegLoad>(field, idx, n, lines, Sp, groups, sms, cyc));
    }
    std::printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
