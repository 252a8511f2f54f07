// K3, level executor (one problem; volumes): mart_level_kernel
//
// The lines of one ASAP dependency level have disjoint supports, so a level is
// one kernel: a small block per line with a non-zero measurement gathers the
// line's cells from its traced list, sums them (fp64), forms the reference's
// factor (mart_update_line, proj/src/solver.cpp:33-51) and scales the cells.
// Levels follow each other in stream order, so every cell sees exactly the
// reference's sequence of updates (solver.cpp:111-136).
//
// What makes a level cost ~3 us instead of a launch gap plus a kernel:
//   * programmatic dependent launch: level l+1 starts while level l runs,
//     loads everything that does not depend on the field (its lines' ids,
//     measurements, list offsets and the lists themselves, into registers),
//     and only then waits for level l (griddepcontrol.wait) — after the wait a
//     block does one gather round trip, a two-warp sum, the factor and its
//     stores;
//   * a 256-thread block per line, three cells a thread held in registers from
//     the sum to the update (measured on C3: 64 / 128 / 256 threads 4.19 /
//     3.78 / 3.47 ms per iteration, 512: 4.04);
//   * lines with a zero measurement (skipped by the reference, solver.cpp:
//     120-124) get no block: per call the level-sorted line order is compacted
//     to the live lines on the device;
//   * a sweep's launches replayed from a CUDA graph that the tracer keeps
//     between calls (plain launches are host-bound at ~2.7 us each; the
//     instantiation costs ~5 us a node, so a graph is built for 16 sweeps or
//     more, or when a call repeats the previous call's buffers and data).
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>
#include <cstdlib>
#include <string>
#include <vector>

#include "internal.cuh"
#include "kernels.h"

namespace ub {

namespace {

template <int NT, int KEEP>
__global__ void __launch_bounds__(NT) mart_level_kernel(const uint32_t* __restrict__ units,
                                                        const unsigned long long* __restrict__ lpos,
                                                        const uint32_t* __restrict__ lists,
                                                        const float* __restrict__ proj, float* __restrict__ f,
                                                        const double* __restrict__ p_floor,
                                                        unsigned long long* clamps, double beta, int power) {
    __shared__ double red[NT / 32];
    // before the wait: nothing here reads the field
    const uint32_t u = units[blockIdx.x];
    const float m = proj[u];
    const double pf = p_floor[0];
    const unsigned long long b = lpos[u];
    const uint32_t n = uint32_t(lpos[u + 1] - b);
    const uint32_t* __restrict__ src = lists + b;
    uint32_t id[KEEP];
    float v[KEEP];
#pragma unroll
    for (int i = 0; i < KEEP; ++i) {
        const uint32_t k = threadIdx.x + uint32_t(i) * NT;
        id[i] = k < n ? __ldcs(src + k) : 0xFFFFFFFFu;
    }
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    // every block waits, also one with nothing to do: a grid must not complete
    // before its predecessor (the next level waits on this grid only)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (m == 0.f)
        return;
#pragma unroll
    for (int i = 0; i < KEEP; ++i)
        v[i] = id[i] != 0xFFFFFFFFu ? __ldcg(f + id[i]) : 0.f;
    double s = 0;
#pragma unroll
    for (int i = 0; i < KEEP; ++i)
        s += double(v[i]);
    for (uint32_t k = threadIdx.x + KEEP * NT; k < n; k += NT)
        s += double(__ldcg(f + __ldcs(src + k)));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        s += __shfl_xor_sync(0xFFFFFFFFu, s, o);
    if ((threadIdx.x & 31) == 0)
        red[threadIdx.x >> 5] = s;
    __syncthreads();
    double p_bar = 0;
#pragma unroll
    for (int k = 0; k < NT / 32; ++k)
        p_bar += red[k];
    // mart_update_line (solver.cpp:36-46)
    const double ratio = double(m) / (p_bar > pf ? p_bar : pf);
    double factor = mart_factor(ratio, beta, power);
    if (factor <= 0) {
        factor = pf;
        if (threadIdx.x == 0)
            atomicAdd(clamps, 1ull);
    }
    // fp32 multiplier; the clamp keeps the fp64 field strictly positive
    // (solver.cpp:42-45): an fp32 product below FLT_MIN saturates there
    const float g = float(factor);
#pragma unroll
    for (int i = 0; i < KEEP; ++i)
        if (id[i] != 0xFFFFFFFFu)
            __stcg(f + id[i], fmaxf(v[i] * g, FLT_MIN));
    for (uint32_t k = threadIdx.x + KEEP * NT; k < n; k += NT) {
        const uint32_t c = __ldcs(src + k);
        __stcg(f + c, fmaxf(__ldcg(f + c) * g, FLT_MIN));
    }
}

__global__ void live_flag_kernel(const uint32_t* __restrict__ order, const float* __restrict__ proj, uint32_t n,
                                 uint32_t* __restrict__ flags) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n)
        flags[k] = proj[order[k]] != 0.f ? 1u : 0u;
}

__global__ void live_compact_kernel(const uint32_t* __restrict__ order, const uint32_t* __restrict__ flags,
                                    const uint32_t* __restrict__ pos, uint32_t n, uint32_t* __restrict__ out) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n && flags[k])
        out[pos[k]] = order[k];
}

__global__ void gather_u32_kernel(const uint32_t* __restrict__ src, const uint32_t* __restrict__ at, uint32_t n,
                                  uint32_t* __restrict__ out) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n)
        out[k] = src[at[k]];
}

}  // namespace

void launch_live_lines(const uint32_t* order, const float* proj, uint32_t units, const uint32_t* level_off_dev,
                       uint32_t levels, uint32_t* flags, uint32_t* pos, uint32_t* live, uint32_t* live_off_dev,
                       cudaStream_t st) {
    if (units == 0)
        return;
    const unsigned blocks = (units + 255) / 256;
    live_flag_kernel<<<blocks, 256, 0, st>>>(order, proj, units, flags);
    launch_exclusive_scan_u32(flags, pos, int(units), st);  // pos[units] = live lines
    live_compact_kernel<<<blocks, 256, 0, st>>>(order, flags, pos, units, live);
    gather_u32_kernel<<<(levels + 1 + 255) / 256, 256, 0, st>>>(pos, level_off_dev, levels + 1, live_off_dev);
    count_launch(3);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        throw CudaError(std::string("live-line compaction launch: ") + cudaGetErrorString(e));
}

void LevelGraphCache::reset() {
    if (exec)
        cudaGraphExecDestroy(exec);
    exec = nullptr;
}

void launch_mart_levels(const MartArgs& h, const LevelSchedule& ls, int sweeps, cudaStream_t st,
                        LevelGraphCache* cache) {
    if (h.Sp != 1)
        throw CudaError("mart_level_kernel runs one problem");
    static const int nt = [] {
        const char* e = std::getenv("USCG_LEVEL_THREADS");
        const int v = e ? std::atoi(e) : 256;
        return v == 128 ? 128 : (v == 64 ? 64 : 256);
    }();
    static const bool pdl = [] {
        const char* e = std::getenv("USCG_LEVEL_PDL");
        return !(e && !std::atoi(e));
    }();
    const int levels = int(ls.live_off.size()) - 1;
    if (levels <= 0 || sweeps <= 0)
        return;
    auto one_sweep = [&] {
        for (int l = 0; l < levels; ++l) {
            const uint32_t n = ls.live_off[l + 1] - ls.live_off[l];
            if (n == 0)
                continue;
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(n);
            cfg.blockDim = dim3(unsigned(nt));
            cfg.stream = st;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = attr;
            cfg.numAttrs = pdl ? 1 : 0;
            const uint32_t* units = ls.live + ls.live_off[l];
            if (nt == 256)
                UB_CUDA(cudaLaunchKernelEx(&cfg, mart_level_kernel<256, 3>, units, ls.lpos, ls.lists, h.proj, h.field,
                                           h.p_floor, h.clamps, h.beta, h.power));
            else if (nt == 128)
                UB_CUDA(cudaLaunchKernelEx(&cfg, mart_level_kernel<128, 6>, units, ls.lpos, ls.lists, h.proj, h.field,
                                           h.p_floor, h.clamps, h.beta, h.power));
            else
                UB_CUDA(cudaLaunchKernelEx(&cfg, mart_level_kernel<64, 12>, units, ls.lpos, ls.lists, h.proj, h.field,
                                           h.p_floor, h.clamps, h.beta, h.power));
        }
    };
    int launched = 0;
    for (int l = 0; l < levels; ++l)
        launched += ls.live_off[l + 1] > ls.live_off[l];
    // Plain launches are issued at ~2.7 us each, about the rate the levels run
    // at (C3: 3.4 ms per iteration, host-bound); a replayed graph runs them at
    // the device's rate (2.9 ms) but costs ~5 us a node to instantiate. So: a
    // cached graph is replayed while its key comes back; a new one is built for
    // 16 sweeps or more, or — after the launches of this call are issued — when
    // the call repeats the key of the call before it.
    const char* ge = std::getenv("USCG_LEVEL_GRAPH");
    const bool allow = launched >= 8 && !(ge && !std::atoi(ge));
    const bool force = ge && std::atoi(ge) != 0 && sweeps >= 2;
    LevelGraphCache local;
    LevelGraphCache* gc = cache ? cache : &local;
    LevelGraphCache::Key key;
    key.field = h.field, key.proj = h.proj, key.p_floor = h.p_floor, key.clamps = h.clamps;
    key.lists = ls.lists, key.lpos = ls.lpos, key.live = ls.live;
    key.beta = h.beta, key.power = h.power, key.threads = nt, key.pdl = pdl ? 1 : 0;
    key.live_off = ls.live_off;
    auto build = [&] {
        cudaGraph_t g = nullptr;
        cudaGraphExec_t exec = nullptr;
        UB_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        try {
            one_sweep();
        } catch (...) {
            cudaStreamEndCapture(st, &g);
            if (g)
                cudaGraphDestroy(g);
            throw;
        }
        UB_CUDA(cudaStreamEndCapture(st, &g));
        const cudaError_t ie = cudaGraphInstantiate(&exec, g, 0);
        cudaGraphDestroy(g);
        UB_CUDA(ie);
        if (gc->exec) {  // the old graph may still be running
            UB_CUDA(cudaStreamSynchronize(st));
            gc->reset();
        }
        gc->exec = exec;
        gc->key = key;
    };
    const bool hit = allow && gc->exec && gc->key == key;
    if (hit || (allow && (force || sweeps >= 16))) {
        if (!hit)
            build();
        for (int s = 0; s < sweeps; ++s)
            UB_CUDA(cudaGraphLaunch(gc->exec, st));
        if (!cache)  // a graph that is not kept must outlive its launches
            UB_CUDA(cudaStreamSynchronize(st));
    } else {
        for (int s = 0; s < sweeps; ++s)
            one_sweep();
        if (allow && cache) {
            if (cache->have_seen && cache->seen == key)
                build();  // the same solve again: the next one replays (built while this one runs)
            cache->seen = key;
            cache->have_seen = true;
        }
    }
    count_launch(uint64_t(launched) * uint64_t(sweeps));
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        throw CudaError(std::string("mart_level_kernel launch: ") + cudaGetErrorString(e));
}

}  // namespace ub
