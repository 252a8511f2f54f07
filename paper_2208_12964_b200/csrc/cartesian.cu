// Cartesian comparator (proj/src/siddon.cpp): the
// paper's baseline, MART on an axis-aligned voxel grid with Siddon path-length
// coefficients, on the device so that the USPG path is compared with it on
// the same hardware.
//
//   siddon_*_kernel   precompute_cartesian_system (siddon.cpp:104-125): one
//                     thread per (view, line) walks the rotated ray through the
//                     voxels (siddon_trace, siddon.cpp:33-102, same fp64
//                     operations in the same order), count pass + write pass
//                     into CSR lists (u32 voxel, f32 length)
//   csr_level_kernel  one dependency level of cartesian_mart_stored
//                     (siddon.cpp:147-165,186-209): block per line, p_bar =
//                     sum w f (fp64), the reference's factor applied to every
//                     crossed voxel
//   otf_level_kernel  cartesian_mart_otf (siddon.cpp:167-184): the same, the
//                     line's Siddon walk recomputed in the block every pass
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>
#include <cstdlib>

#include "kernels.h"

namespace ub {

namespace {
constexpr double kRadPerDegC = 3.141592653589793238462643383279502884 / 180.0;
constexpr int kLevelThreads = 256;

// rotate_z_deg (scan.cpp:50-54) of the first-view endpoints of `line`
__device__ __forceinline__ void rotated_ray(const double* rays, int lines, int line, double theta_deg,
                                            double* s, double* d) {
    const double rad = theta_deg * kRadPerDegC;
    const double c = cos(rad), sn = sin(rad);
    const double* s0 = rays + 3 * size_t(line);
    const double* d0 = rays + 3 * (size_t(lines) + line);
    s[0] = c * s0[0] - sn * s0[1];
    s[1] = sn * s0[0] + c * s0[1];
    s[2] = s0[2];
    d[0] = c * d0[0] - sn * d0[1];
    d[1] = sn * d0[0] + c * d0[1];
    d[2] = d0[2];
}

// siddon_trace (siddon.cpp:33-102): every crossed voxel with its chord length
template <class Emit>
__device__ void siddon_walk(const double* s, const double* d, const DevCart& C, Emit&& emit) {
    const double dir[3] = {d[0] - s[0], d[1] - s[1], d[2] - s[2]};
    const double lo[3] = {C.o0, C.o1, C.o2};
    const int count[3] = {C.nx, C.ny, C.nz};
    const double length = sqrt(dir[0] * dir[0] + dir[1] * dir[1] + dir[2] * dir[2]);
    if (length == 0)
        return;
    double tau_min = 0.0, tau_max = 1.0;
    for (int a = 0; a < 3; ++a) {
        const double hi = lo[a] + count[a] * C.voxel;
        if (dir[a] == 0) {
            if (s[a] < lo[a] || s[a] > hi)
                return;
            continue;
        }
        double t0 = (lo[a] - s[a]) / dir[a];
        double t1 = (hi - s[a]) / dir[a];
        if (t0 > t1) {
            const double t = t0;
            t0 = t1;
            t1 = t;
        }
        tau_min = fmax(tau_min, t0);
        tau_max = fmin(tau_max, t1);
    }
    if (tau_min >= tau_max)
        return;
    int vox[3], step[3];
    double next[3], delta[3];
    for (int a = 0; a < 3; ++a) {
        const double entry = s[a] + tau_min * dir[a];
        int i = int(floor((entry - lo[a]) / C.voxel));
        i = i < 0 ? 0 : (i > count[a] - 1 ? count[a] - 1 : i);
        vox[a] = i;
        if (dir[a] == 0) {
            step[a] = 0;
            delta[a] = 0;
            next[a] = __longlong_as_double(0x7FF0000000000000LL);  // +inf
        } else {
            step[a] = dir[a] > 0 ? 1 : -1;
            delta[a] = C.voxel / fabs(dir[a]);
            const double boundary = lo[a] + (i + (dir[a] > 0 ? 1 : 0)) * C.voxel;
            next[a] = (boundary - s[a]) / dir[a];
        }
    }
    double tau = tau_min;
    while (true) {
        int axis = 0;
        if (next[1] < next[axis])
            axis = 1;
        if (next[2] < next[axis])
            axis = 2;
        const double tau_next = fmin(next[axis], tau_max);
        if (tau_next > tau)
            emit(uint32_t((uint32_t(vox[2]) * uint32_t(C.ny) + uint32_t(vox[1])) * uint32_t(C.nx) +
                          uint32_t(vox[0])),
                 (tau_next - tau) * length);
        if (tau_next >= tau_max)
            break;
        vox[axis] += step[axis];
        if (vox[axis] < 0 || vox[axis] >= count[axis])
            break;
        next[axis] += delta[axis];
        tau = tau_next;
    }
}

template <int NT = kLevelThreads>
__device__ __forceinline__ double block_sum_d(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    if ((threadIdx.x & 31) == 0)
        red[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0;
#pragma unroll
    for (int k = 0; k < NT / 32; ++k)
        s += red[k];
    return s;  // every thread
}

// the reference's factor (siddon.cpp:152-164) as an fp32 multiplier; -1 = no update
__device__ __forceinline__ float cart_factor(double p_bar, double m, double beta, double p_floor,
                                             unsigned long long* clamps) {
    if (m == 0)
        return -1.f;
    const double ratio = m / (p_bar > p_floor ? p_bar : p_floor);
    double factor = 1.0 - beta * (1.0 - ratio);
    if (factor <= 0) {
        factor = p_floor;
        if (threadIdx.x == 0)
            atomicAdd(clamps, 1ull);
    }
    return float(factor);
}
}  // namespace

__global__ void siddon_count_kernel(DevCart C, int lines, int views, const double* __restrict__ rays,
                                    const double* __restrict__ theta, uint32_t* __restrict__ counts) {
    const long long u = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= (long long)lines * views)
        return;
    double s[3], d[3];
    rotated_ray(rays, lines, int(u % lines), theta[u / lines], s, d);
    uint32_t n = 0;
    siddon_walk(s, d, C, [&](uint32_t, double) { ++n; });
    counts[u] = n;
}

__global__ void siddon_write_kernel(DevCart C, int lines, int views, const double* __restrict__ rays,
                                    const double* __restrict__ theta, const uint32_t* __restrict__ off,
                                    uint32_t* __restrict__ idx, float* __restrict__ w) {
    const long long u = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= (long long)lines * views)
        return;
    double s[3], d[3];
    rotated_ray(rays, lines, int(u % lines), theta[u / lines], s, d);
    uint32_t k = off[u];
    siddon_walk(s, d, C, [&](uint32_t v, double len) {
        idx[k] = v;
        w[k] = float(len);
        ++k;
    });
}

// stored coefficients: block per line of the level. NT threads hold KEEP
// entries each in registers from the sum to the update (a polar line holds a
// few hundred cells: all of them); small blocks, so that a level's lines and
// the next level's waiting blocks are resident together.
template <int NT, int KEEP>
__global__ void __launch_bounds__(NT) csr_level_kernel(
    const uint32_t* __restrict__ units, const uint32_t* __restrict__ off, const uint32_t* __restrict__ idx,
    const float* __restrict__ w, const float* __restrict__ proj, float* __restrict__ f, double beta,
    double p_floor, unsigned long long* clamps) {
    __shared__ double red[NT / 32];
    // Programmatic dependent launch: this grid may start while the previous
    // level still runs. Everything that does not depend on the field (the
    // line's measurement, offsets, indices and lengths) is loaded first; the
    // next level is released to do the same; then the grid waits for the
    // previous level's completion (and its stores) before touching the field.
    // Every block waits, also one that has nothing to do: a grid must not
    // complete before its predecessor (the level after it waits on this grid
    // only).
    const uint32_t u = units[blockIdx.x];
    const float m = proj[u];
    uint32_t id[KEEP];
    float wk[KEEP], v[KEEP];
    uint32_t b = 0, e = 0;
    if (m != 0.f) {  // weighted_update (siddon.cpp:143): a zero measurement is skipped, nothing read
        b = off[u];
        e = off[u + 1];
    }
#pragma unroll
    for (int i = 0; i < KEEP; ++i) {
        const uint32_t k = b + threadIdx.x + uint32_t(i) * NT;
        id[i] = k < e ? idx[k] : 0xFFFFFFFFu;
        wk[i] = k < e ? w[k] : 0.f;
    }
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (m == 0.f)
        return;
    double s = 0;
#pragma unroll
    for (int i = 0; i < KEEP; ++i)
        v[i] = id[i] != 0xFFFFFFFFu ? __ldcg(f + id[i]) : 0.f;
#pragma unroll
    for (int i = 0; i < KEEP; ++i)
        s += double(wk[i]) * double(v[i]);
    for (uint32_t k = b + threadIdx.x + KEEP * NT; k < e; k += NT)
        s += double(w[k]) * double(__ldcg(f + idx[k]));
    const double p_bar = block_sum_d<NT>(s, red);
    const float g = cart_factor(p_bar, m, beta, p_floor, clamps);
    if (g < 0.f)
        return;
#pragma unroll
    for (int i = 0; i < KEEP; ++i)
        if (id[i] != 0xFFFFFFFFu)
            f[id[i]] = fmaxf(v[i] * g, FLT_MIN);
    for (uint32_t k = b + threadIdx.x + KEEP * NT; k < e; k += NT)
        f[idx[k]] = fmaxf(__ldcg(f + idx[k]) * g, FLT_MIN);
}

// on the fly: thread 0 walks the line into shared memory, then the block updates
__global__ void __launch_bounds__(kLevelThreads) otf_level_kernel(
    DevCart C, int lines, const double* __restrict__ rays, const double* __restrict__ theta,
    const uint32_t* __restrict__ units, const float* __restrict__ proj, float* __restrict__ f, double beta,
    double p_floor, unsigned long long* clamps) {
    extern __shared__ uint32_t s_idx[];  // [cap] voxels then [cap] lengths (f32)
    __shared__ double red[kLevelThreads / 32];
    __shared__ uint32_t s_n;
    const int cap = C.nx + C.ny + C.nz + 3;
    float* s_w = reinterpret_cast<float*>(s_idx + cap);
    const uint32_t u = units[blockIdx.x];
    if (threadIdx.x == 0) {
        double s[3], d[3];
        rotated_ray(rays, lines, int(u % uint32_t(lines)), theta[u / uint32_t(lines)], s, d);
        uint32_t n = 0;
        siddon_walk(s, d, C, [&](uint32_t v, double len) {
            s_idx[n] = v;
            s_w[n] = float(len);
            ++n;
        });
        s_n = n;
    }
    __syncthreads();
    const uint32_t n = s_n;
    double acc = 0;
    for (uint32_t k = threadIdx.x; k < n; k += kLevelThreads)
        acc += double(s_w[k]) * double(f[s_idx[k]]);
    const double p_bar = block_sum_d(acc, red);
    const float g = cart_factor(p_bar, proj[u], beta, p_floor, clamps);
    if (g < 0.f)
        return;
    for (uint32_t k = threadIdx.x; k < n; k += kLevelThreads)
        f[s_idx[k]] = fmaxf(f[s_idx[k]] * g, FLT_MIN);
}

void launch_siddon_count(const DevCart& C, int lines, int views, const double* rays, const double* theta,
                         uint32_t* counts, cudaStream_t st) {
    const long long units = (long long)lines * views;
    if (units <= 0)
        return;
    siddon_count_kernel<<<unsigned((units + 127) / 128), 128, 0, st>>>(C, lines, views, rays, theta, counts);
    count_launch();
    UB_CUDA(cudaGetLastError());
}

void launch_siddon_write(const DevCart& C, int lines, int views, const double* rays, const double* theta,
                         const uint32_t* off, uint32_t* idx, float* w, cudaStream_t st) {
    const long long units = (long long)lines * views;
    if (units <= 0)
        return;
    siddon_write_kernel<<<unsigned((units + 127) / 128), 128, 0, st>>>(C, lines, views, rays, theta, off, idx, w);
    count_launch();
    UB_CUDA(cudaGetLastError());
}

void launch_csr_level(const uint32_t* units, int n, const uint32_t* off, const uint32_t* idx, const float* w,
                      const float* proj, float* f, double beta, double p_floor, unsigned long long* clamps,
                      cudaStream_t st) {
    if (n <= 0)
        return;
    // launched with programmatic stream serialization (the kernel orders itself
    // after the previous level with griddepcontrol.wait); USCG_CSR_PDL=0: plain
    static const bool pdl = [] {
        const char* e = std::getenv("USCG_CSR_PDL");
        return !(e && !std::atoi(e));
    }();
    // threads per line (USCG_CSR_THREADS = 64 | 128 | 256; default 128)
    static const int nt = [] {
        const char* e = std::getenv("USCG_CSR_THREADS");
        const int v = e ? std::atoi(e) : 128;
        return v == 256 ? 256 : (v == 64 ? 64 : 128);
    }();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(n));
    cfg.blockDim = dim3(unsigned(nt));
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    if (nt == 256)
        UB_CUDA(cudaLaunchKernelEx(&cfg, csr_level_kernel<256, 4>, units, off, idx, w, proj, f, beta, p_floor, clamps));
    else if (nt == 128)
        UB_CUDA(cudaLaunchKernelEx(&cfg, csr_level_kernel<128, 6>, units, off, idx, w, proj, f, beta, p_floor, clamps));
    else
        UB_CUDA(cudaLaunchKernelEx(&cfg, csr_level_kernel<64, 8>, units, off, idx, w, proj, f, beta, p_floor, clamps));
    count_launch();
}

void launch_otf_level(const DevCart& C, int lines, const double* rays, const double* theta, const uint32_t* units,
                      int n, const float* proj, float* f, double beta, double p_floor, unsigned long long* clamps,
                      cudaStream_t st) {
    if (n <= 0)
        return;
    const size_t sm = sizeof(uint32_t) * 2 * size_t(C.nx + C.ny + C.nz + 3);
    otf_level_kernel<<<unsigned(n), kLevelThreads, sm, st>>>(C, lines, rays, theta, units, proj, f, beta, p_floor,
                                                             clamps);
    count_launch();
}

}  // namespace ub
