// Image-quality metrics on the device (proj/src/metrics.cpp): per-slice MAE,
// RMSE and SSIM of a stack of rows x cols rasters (fp32 in, fp64 arithmetic),
// for the reference's volume scores (mae/rmse/ssim_volume, metrics.cpp:170-199).
//
// SSIM (metrics.cpp:62-136): 8x8 windows at stride 1, C1 = (0.01 L)^2,
// C2 = (0.03 L)^2. A block scores a 16 x 32 tile of window origins from a
// 23 x 39 pixel tile in shared memory: five moments (x, y, xx, yy, xy) summed
// over 8 columns, then over 8 rows (separable box sums; the reference sums
// the 64 terms row-major, a different fp64 order, ~1 ulp). Per-block partial
// sums are reduced in a fixed order (deterministic, no fp64 atomics).
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>

#include "kernels.h"

namespace ub {

namespace {
constexpr int kWin = 8;
constexpr int kTileR = 16, kTileC = 32;  // window origins per tile (rows x cols)
constexpr int kPixR = kTileR + kWin - 1, kPixC = kTileC + kWin - 1;  // pixels per tile
constexpr int kThreads = 256;

__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0)
        red[w] = v;
    __syncthreads();
    double s = 0;
    if (threadIdx.x == 0)
        for (int k = 0; k < kThreads / 32; ++k)
            s += red[k];
    return s;  // valid in thread 0
}
}  // namespace

// per slice: [0] min of ref, [1] max of ref, [2] sum |ref - test|, [3] sum (ref - test)^2
// (per-block partials; blockIdx.y = slice)
__global__ void __launch_bounds__(kThreads) moments_kernel(const float* __restrict__ ref,
                                                           const float* __restrict__ test, uint64_t px,
                                                           double* __restrict__ part) {
    __shared__ double red[kThreads / 32];
    const size_t s = blockIdx.y;
    const float* a = ref + s * px;
    const float* b = test + s * px;
    double lo = DBL_MAX, hi = -DBL_MAX, sa = 0, sq = 0;
    for (uint64_t i = uint64_t(blockIdx.x) * kThreads + threadIdx.x; i < px; i += uint64_t(gridDim.x) * kThreads) {
        const double x = a[i], d = x - double(b[i]);
        lo = fmin(lo, x);
        hi = fmax(hi, x);
        sa += fabs(d);
        sq += d * d;
    }
    // min / max through the sum reduction's scratch, one quantity at a time
    __shared__ double mm[2][kThreads / 32];
    double l = lo, h = hi;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        l = fmin(l, __shfl_xor_sync(0xFFFFFFFFu, l, o));
        h = fmax(h, __shfl_xor_sync(0xFFFFFFFFu, h, o));
    }
    if ((threadIdx.x & 31) == 0) {
        mm[0][threadIdx.x >> 5] = l;
        mm[1][threadIdx.x >> 5] = h;
    }
    const double tsa = block_sum(sa, red);
    const double tsq = block_sum(sq, red);
    if (threadIdx.x == 0) {
        for (int k = 0; k < kThreads / 32; ++k) {
            l = fmin(l, mm[0][k]);
            h = fmax(h, mm[1][k]);
        }
        double* p = part + (s * gridDim.x + blockIdx.x) * 4;
        p[0] = l;
        p[1] = h;
        p[2] = tsa;
        p[3] = tsq;
    }
}

// sum over the windows of one tile: blockIdx.x = tile, blockIdx.y = slice.
// c1c2: [slice][2] (per-slice constants from the dynamic range)
__global__ void __launch_bounds__(kThreads) ssim_kernel(const float* __restrict__ ref,
                                                        const float* __restrict__ test, int rows,
                                                        int cols, const double* __restrict__ c1c2,
                                                        double* __restrict__ part) {
    __shared__ float sx[kPixR][kPixC + 1], sy[kPixR][kPixC + 1];
    __shared__ double h[5][kPixR][kTileC];
    __shared__ double red[kThreads / 32];
    const size_t s = blockIdx.y;
    const int wr = rows - kWin + 1, wc = cols - kWin + 1;  // window origins
    const int tiles_c = (wc + kTileC - 1) / kTileC;
    const int r0 = (int(blockIdx.x) / tiles_c) * kTileR, c0 = (int(blockIdx.x) % tiles_c) * kTileC;
    const float* a = ref + s * size_t(rows) * cols;
    const float* b = test + s * size_t(rows) * cols;
    for (int k = threadIdx.x; k < kPixR * kPixC; k += kThreads) {
        const int r = r0 + k / kPixC, c = c0 + k % kPixC;
        const bool in = r < rows && c < cols;
        sx[k / kPixC][k % kPixC] = in ? a[size_t(r) * cols + c] : 0.f;
        sy[k / kPixC][k % kPixC] = in ? b[size_t(r) * cols + c] : 0.f;
    }
    __syncthreads();
    // horizontal 8-sums of the five moments for every tile row
    for (int k = threadIdx.x; k < kPixR * kTileC; k += kThreads) {
        const int r = k / kTileC, c = k % kTileC;
        double m0 = 0, m1 = 0, m2 = 0, m3 = 0, m4 = 0;
#pragma unroll
        for (int j = 0; j < kWin; ++j) {
            const double x = sx[r][c + j], y = sy[r][c + j];
            m0 += x;
            m1 += y;
            m2 += x * x;
            m3 += y * y;
            m4 += x * y;
        }
        h[0][r][c] = m0;
        h[1][r][c] = m1;
        h[2][r][c] = m2;
        h[3][r][c] = m3;
        h[4][r][c] = m4;
    }
    __syncthreads();
    const double c1 = c1c2[2 * s], c2 = c1c2[2 * s + 1];
    constexpr double inv_n = 1.0 / (kWin * kWin);
    double acc = 0;
    for (int k = threadIdx.x; k < kTileR * kTileC; k += kThreads) {
        const int r = k / kTileC, c = k % kTileC;
        if (r0 + r >= wr || c0 + c >= wc)
            continue;
        double m[5] = {0, 0, 0, 0, 0};
#pragma unroll
        for (int j = 0; j < kWin; ++j)
#pragma unroll
            for (int q = 0; q < 5; ++q)
                m[q] += h[q][r + j][c];
        const double mx = m[0] * inv_n, my = m[1] * inv_n;
        const double vx = m[2] * inv_n - mx * mx, vy = m[3] * inv_n - my * my;
        const double cov = m[4] * inv_n - mx * my;
        acc += ((2 * mx * my + c1) * (2 * cov + c2)) / ((mx * mx + my * my + c1) * (vx + vy + c2));
    }
    const double t = block_sum(acc, red);
    if (threadIdx.x == 0)
        part[s * gridDim.x + blockIdx.x] = t;
}

// per slice, in block order: moments partials -> [min, max, sum|d|, sum d^2]
__global__ void fold_moments_kernel(const double* __restrict__ part, int blocks, int slices,
                                    double* __restrict__ out) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= slices)
        return;
    double lo = DBL_MAX, hi = -DBL_MAX, sa = 0, sq = 0;
    for (int k = 0; k < blocks; ++k) {
        const double* p = part + (size_t(s) * blocks + k) * 4;
        lo = fmin(lo, p[0]);
        hi = fmax(hi, p[1]);
        sa += p[2];
        sq += p[3];
    }
    out[4 * s + 0] = lo;
    out[4 * s + 1] = hi;
    out[4 * s + 2] = sa;
    out[4 * s + 3] = sq;
}

__global__ void fold_ssim_kernel(const double* __restrict__ part, int tiles, int slices,
                                 double windows, double* __restrict__ out) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= slices)
        return;
    double acc = 0;
    for (int k = 0; k < tiles; ++k)
        acc += part[size_t(s) * tiles + k];
    out[s] = acc / windows;
}

int metrics_blocks(uint64_t px) {
    const uint64_t b = (px + kThreads * 8 - 1) / (kThreads * 8);
    return int(b < 1 ? 1 : (b > 1024 ? 1024 : b));
}

void launch_moments(const float* ref, const float* test, int slices, uint64_t px, double* part,
                    double* out, cudaStream_t st) {
    const int nb = metrics_blocks(px);
    moments_kernel<<<dim3(nb, slices), kThreads, 0, st>>>(ref, test, px, part);
    count_launch();
    fold_moments_kernel<<<(slices + 127) / 128, 128, 0, st>>>(part, nb, slices, out);
    count_launch();
    UB_CUDA(cudaGetLastError());
}

// sharpness (metrics.cpp:138-152): per pixel the central-difference gradient
// magnitude, one-sided at the borders (the clamped neighbours, divided by
// their distance), fp64 from the fp32 raster; per-block partial sums of one
// slice (blockIdx.y), folded in block order
__global__ void __launch_bounds__(kThreads) sharpness_kernel(const float* __restrict__ img, int rows, int cols,
                                                             double* __restrict__ part) {
    __shared__ double red[kThreads / 32];
    const uint64_t px = uint64_t(rows) * uint64_t(cols);
    const float* a = img + size_t(blockIdx.y) * px;
    double acc = 0;
    for (uint64_t i = uint64_t(blockIdx.x) * kThreads + threadIdx.x; i < px; i += uint64_t(gridDim.x) * kThreads) {
        const int r = int(i / uint64_t(cols)), c = int(i % uint64_t(cols));
        const int cl = c > 0 ? c - 1 : 0, ch = c + 1 < cols ? c + 1 : cols - 1;
        const int rl = r > 0 ? r - 1 : 0, rh = r + 1 < rows ? r + 1 : rows - 1;
        const double gx = (double(a[size_t(r) * cols + ch]) - double(a[size_t(r) * cols + cl])) / double(ch - cl);
        const double gy = (double(a[size_t(rh) * cols + c]) - double(a[size_t(rl) * cols + c])) / double(rh - rl);
        acc += sqrt(gx * gx + gy * gy);
    }
    const double t = block_sum(acc, red);
    if (threadIdx.x == 0)
        part[size_t(blockIdx.y) * gridDim.x + blockIdx.x] = t;
}

__global__ void fold_mean_kernel(const double* __restrict__ part, int blocks, int slices, double n,
                                 double* __restrict__ out) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= slices)
        return;
    double acc = 0;
    for (int k = 0; k < blocks; ++k)
        acc += part[size_t(s) * blocks + k];
    out[s] = acc / n;
}

void launch_sharpness(const float* img, int slices, int rows, int cols, double* part, double* out,
                      cudaStream_t st) {
    const uint64_t px = uint64_t(rows) * uint64_t(cols);
    const int nb = metrics_blocks(px);
    sharpness_kernel<<<dim3(nb, slices), kThreads, 0, st>>>(img, rows, cols, part);
    count_launch();
    fold_mean_kernel<<<(slices + 127) / 128, 128, 0, st>>>(part, nb, slices, double(px), out);
    count_launch();
    UB_CUDA(cudaGetLastError());
}

int ssim_tiles(int rows, int cols) {
    const int wr = rows - kWin + 1, wc = cols - kWin + 1;
    return ((wr + kTileR - 1) / kTileR) * ((wc + kTileC - 1) / kTileC);
}

void launch_ssim(const float* ref, const float* test, int slices, int rows, int cols,
                 const double* c1c2, double* part, double* out, cudaStream_t st) {
    const int tiles = ssim_tiles(rows, cols);
    ssim_kernel<<<dim3(tiles, slices), kThreads, 0, st>>>(ref, test, rows, cols, c1c2, part);
    count_launch();
    const double windows = double(rows - kWin + 1) * double(cols - kWin + 1);
    fold_ssim_kernel<<<(slices + 127) / 128, 128, 0, st>>>(part, tiles, slices, windows, out);
    count_launch();
    UB_CUDA(cudaGetLastError());
}

}  // namespace ub
