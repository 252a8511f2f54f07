// K3 for one small problem: the whole Sp-MART reconstruction in one CTA with
// the field in shared memory ("Config 1 (51 KB field) runs as a
// single CTA with the field in shared memory and __syncthreads between
// levels").
//
// The reference's row action (proj/src/solver.cpp:111-136) is replayed level
// by level: the lines of one ASAP dependency level have pairwise disjoint
// cell supports (their updates commute), so each warp applies one line of the
// level to the shared-memory field, and a block barrier separates levels.
// Every cell therefore sees exactly the reference's sequence of updates.
// The per-line work is the reference's: p̄ = Σ f over the line's active cells
// (solver.cpp:25-31, fp64), factor = 1 − β(1 − m / max(p̄, p_floor)) with the
// clamp and the zero-measurement skip (solver.cpp:33-51), f *= factor.
//
// Each line's traced index list comes from the precomputed lists in global
// memory (L2-resident for these sizes); a warp loads the lists of its lines
// two levels ahead into registers, so the loads' latency overlaps the two
// levels before. The per-line metadata, measurements and level offsets are
// staged in shared memory with the field.
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "kernels.h"

namespace ub {

namespace {
constexpr int kTileNT = 512;  // 16 line warps: registers for three prefetched lists per lane
constexpr int kTileW = kTileNT / 32;
constexpr int kTileK = 8;  // prefetched cells per lane: lines of up to 256 cells (longer: direct loads)

struct TileKernelArgs {
    MartArgs m;
    TileSchedule ts;
    int sweeps;
    uint32_t cells;
};

__host__ __device__ inline size_t round4w(size_t w) { return (w + 3) & ~size_t(3); }

// shared memory: meta [units] uint4 | measurements [units] f32 | level offsets
// [levels + 1] u32 | field [cells] f32 (all 16-byte aligned)
__host__ __device__ inline size_t tile_words(uint64_t cells, int units, int levels) {
    return 4 * size_t(units) + round4w(size_t(units)) + round4w(size_t(levels) + 1) + round4w(size_t(cells));
}

// a line's prefetched state: its metadata, measurement and index list
struct TileLine {
    uint32_t idx[kTileK];
    uint32_t off, n;
    float m;
    int slot;  // -1: none
};

__device__ __forceinline__ void fetch(const TileSchedule& ts, const uint4* s_meta, const float* s_m, int slot,
                                      int lane, TileLine& r) {
    r.slot = slot;
    if (slot < 0)
        return;
    const uint4 md = s_meta[slot];
    r.off = md.y;
    r.n = md.z;
    r.m = s_m[slot];
#pragma unroll
    for (int i = 0; i < kTileK; ++i) {
        const uint32_t k = uint32_t(lane + 32 * i);
        r.idx[i] = k < md.z ? __ldg(ts.lists + md.y + k) : 0u;
    }
}

__global__ void __launch_bounds__(kTileNT, 1) mart_tile_kernel(TileKernelArgs a) {
    extern __shared__ __align__(16) uint32_t smem[];
    const TileSchedule& ts = a.ts;
    const int units = ts.units, levels = ts.levels;
    uint4* s_meta = reinterpret_cast<uint4*>(smem);
    float* s_m = reinterpret_cast<float*>(smem + 4 * size_t(units));
    uint32_t* s_lo = reinterpret_cast<uint32_t*>(s_m + round4w(size_t(units)));
    float* s_f = reinterpret_cast<float*>(s_lo + round4w(size_t(levels) + 1));
    const int tid = int(threadIdx.x), lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < units; i += kTileNT) {
        const uint4 md = ts.meta[i];
        s_meta[i] = md;
        s_m[i] = __ldg(a.m.proj + md.x);
    }
    for (int i = tid; i <= levels; i += kTileNT)
        s_lo[i] = __ldg(ts.level_off + i);
    for (uint32_t c = uint32_t(tid); c < a.cells; c += kTileNT)
        s_f[c] = a.m.field[c];
    __syncthreads();
    const double beta = a.m.beta, pf = a.m.p_floor[0];
    const bool act = a.m.active[0] != 0;
    unsigned long long clamps = 0;
    const int total = a.sweeps * levels;
    // this warp's first slot of global level g (sweep-major), or -1
    auto slot_of = [&](int g) -> int {
        if (g >= total)
            return -1;
        const int L = g % levels;
        const int s = int(s_lo[L]) + warp;
        return s < int(s_lo[L + 1]) ? s : -1;
    };
    // one line of the level: gather, sum, factor, scale (solver.cpp:25-51).
    // The cells' values stay in registers between the sum and the update.
    auto line = [&](const TileLine& r) {
        if (r.m == 0.f || !act)
            return;  // zero-measurement skip (counted by the caller's U/skip counters)
        const uint32_t n = r.n;
        float v[kTileK];
        float ps = 0.f;
#pragma unroll
        for (int i = 0; i < kTileK; ++i) {
            v[i] = uint32_t(lane + 32 * i) < n ? s_f[r.idx[i]] : 0.f;
            ps += v[i];
        }
        // fp32 partials per lane and across the warp's lanes (a line's at
        // most a few hundred cells: relative error ~1e-7, below the field's
        // own fp32 rounding per update), fp64 from the factor on (the
        // reference sums in fp64, solver.cpp:25-31)
        for (uint32_t k = uint32_t(lane + 32 * kTileK); k < n; k += 32)
            ps += s_f[__ldg(ts.lists + r.off + k)];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
            ps += __shfl_xor_sync(0xFFFFFFFFu, ps, o);
        const double s = ps;
        const double ratio = double(r.m) / (s > pf ? s : pf);
        double f = mart_factor(ratio, beta, a.m.power);
        if (f <= 0) {
            f = pf;
            clamps += lane == 0;
        }
        const float g = float(f);
#pragma unroll
        for (int i = 0; i < kTileK; ++i)
            if (uint32_t(lane + 32 * i) < n)
                s_f[r.idx[i]] = fmaxf(v[i] * g, FLT_MIN);
        for (uint32_t k = uint32_t(lane + 32 * kTileK); k < n; k += 32) {
            const uint32_t c = __ldg(ts.lists + r.off + k);
            s_f[c] = fmaxf(s_f[c] * g, FLT_MIN);
        }
    };
    // three line buffers in fixed roles (unrolled by 3): a buffer is read
    // two levels after its loads were issued and never moved (a move would
    // wait for the loads at once)
    TileLine rA, rB, rC;
    int gL = 0;  // level index within the sweep of global level g (no modulo per level)
    auto level = [&](int g, const TileLine& cur, TileLine& ahead) {
        const int b = int(s_lo[gL]), e = int(s_lo[gL + 1]);
        if (cur.slot >= 0)
            line(cur);
        for (int s = b + warp + kTileW; s < e; s += kTileW) {  // levels wider than the CTA's warps
            TileLine rx;
            fetch(ts, s_meta, s_m, s, lane, rx);
            line(rx);
        }
        // the line two levels ahead, issued after this level's line so that
        // its address chain is off this level's path
        int L2 = gL + 2, g2 = g + 2;
        if (L2 >= levels)
            L2 -= levels;
        int s2 = -1;
        if (g2 < total) {
            s2 = int(s_lo[L2]) + warp;
            if (s2 >= int(s_lo[L2 + 1]))
                s2 = -1;
        }
        fetch(ts, s_meta, s_m, s2, lane, ahead);
        if (++gL == levels)
            gL = 0;
        __syncthreads();
    };
    fetch(ts, s_meta, s_m, slot_of(0), lane, rA);
    fetch(ts, s_meta, s_m, slot_of(1), lane, rB);
    for (int g = 0; g < total; g += 3) {
        level(g, rA, rC);
        if (g + 1 < total)
            level(g + 1, rB, rA);
        if (g + 2 < total)
            level(g + 2, rC, rB);
    }
    for (uint32_t c = uint32_t(tid); c < a.cells; c += kTileNT)
        a.m.field[c] = s_f[c];
    if (lane == 0 && clamps)
        atomicAdd(a.m.clamps, clamps);
}
}  // namespace

size_t tile_smem_bytes(uint64_t cells, int units, int levels) { return 4 * tile_words(cells, units, levels); }

bool tile_fits(uint64_t cells, int units, int levels) {
    int optin = 0, dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
        return false;
    return tile_smem_bytes(cells, units, levels) + 64 <= size_t(optin);
}

void launch_mart_tile(const MartArgs& h, const TileSchedule& ts, uint64_t cells, int sweeps, cudaStream_t st) {
    if (h.Sp != 1)
        throw CudaError("mart_tile_kernel: one problem only");
    const size_t smem = tile_smem_bytes(cells, ts.units, ts.levels);
    UB_CUDA(cudaFuncSetAttribute(mart_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    TileKernelArgs a{h, ts, sweeps, uint32_t(cells)};
    if (const char* e = std::getenv("USCG_FLOW_VERBOSE"); e && std::atoi(e))
        std::fprintf(stderr, "mart_tile_kernel: cells=%llu units=%d levels=%d sweeps=%d smem=%zu\n",
                     (unsigned long long)cells, ts.units, ts.levels, sweeps, smem);
    mart_tile_kernel<<<1, kTileNT, smem, st>>>(a);
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        throw CudaError(std::string("mart_tile_kernel launch: ") + cudaGetErrorString(e));
}

}  // namespace ub
