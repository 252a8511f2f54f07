// The MART dependency schedule (schedule.h) built on the device.
//
// The host AsapSchedule walks every traced cell of every line in sweep order,
// keeping the last writer of each cell: one random access per (line, cell)
// visit, 157 s for the C4 volume. The same DAG falls out of a sort: emit one
// key (cell, line) per visit (line = view * lines + detector line is the sweep
// order), radix-sort the keys, and read the edges off consecutive entries:
//   * in-sweep: consecutive visits of one cell from different runs give
//     (earlier run -> later run); a cell's visits by one run are contiguous
//     because a run is a contiguous block of lines;
//   * cross-sweep: a cell's first visitor in a sweep waits for the cell's last
//     visitor of the previous sweep (self edges included, as schedule.cpp).
// Keys are processed in cell ranges sized to the device memory budget; edges
// are deduplicated per range and again at the end. The host then forms the
// CSR lists, the ASAP levels (one pass in run order, which is topological)
// and the level-sorted order, exactly as AsapSchedule does.
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <cstdint>
#include <vector>

#include "kernels.h"

namespace ub {

namespace {
constexpr uint32_t kCross = 0x80000000u;  // flag in an edge's predecessor word
constexpr int kNT = 128;

// a growable raw device buffer
struct Scratch {
    void* p = nullptr;
    size_t bytes = 0;
    void ensure(size_t b) {
        if (b <= bytes)
            return;
        if (p)
            cudaFree(p);
        p = nullptr;
        bytes = 0;
        UB_CUDA(cudaMalloc(&p, b));
        bytes = b;
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
    ~Scratch() {
        if (p)
            cudaFree(p);
    }
};

__device__ __forceinline__ uint32_t run_of(uint32_t u, uint32_t lines, uint32_t run, uint32_t runs_per_view) {
    return (u / lines) * runs_per_view + (u % lines) / run;
}

// block per (view, line): trace, then append (cell - c0, unit) for cells in [c0, c1)
__global__ void __launch_bounds__(kNT) emit_pairs_kernel(TraceArgs A, int max_recs, uint32_t unit0, uint64_t c0,
                                                         uint64_t c1, unsigned long long* __restrict__ keys,
                                                         unsigned long long cap, unsigned long long* __restrict__ n) {
    extern __shared__ uint32_t smem[];
    const TraceSmem S = carve_trace_smem<kNT>(smem, max_recs);
    const uint32_t unit = unit0 + blockIdx.x;
    const int v = int(unit / uint32_t(A.lines)), line = int(unit % uint32_t(A.lines));
    const int cnt = block_trace<kNT>(A, line, A.theta[v], S, true);
    for (int i = threadIdx.x; i < cnt; i += kNT) {
        const uint64_t c = S.idx[i];
        if (c < c0 || c >= c1)
            continue;
        const unsigned long long at = atomicAdd(n, 1ull);
        if (at < cap)
            keys[at] = ((c - c0) << 32) | unit;
    }
}

// edges from the sorted (cell, unit) keys
__global__ void edges_kernel(const unsigned long long* __restrict__ keys, unsigned long long nkeys, uint32_t lines,
                             uint32_t run, uint32_t runs_per_view, unsigned long long* __restrict__ edges,
                             unsigned long long cap, unsigned long long* __restrict__ n) {
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < nkeys;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long k = keys[i];
        const uint32_t cell = uint32_t(k >> 32);
        const uint32_t r = run_of(uint32_t(k), lines, run, runs_per_view);
        if (i > 0 && uint32_t(keys[i - 1] >> 32) == cell) {
            const uint32_t rp = run_of(uint32_t(keys[i - 1]), lines, run, runs_per_view);
            if (rp != r) {
                const unsigned long long at = atomicAdd(n, 1ull);
                if (at < cap)
                    edges[at] = ((unsigned long long)r << 32) | rp;
            }
        }
        if (i + 1 == nkeys || uint32_t(keys[i + 1] >> 32) != cell) {
            // the cell's first visitor waits for this (its last) visitor of the previous sweep
            unsigned long long j = i;
            while (j > 0 && uint32_t(keys[j - 1] >> 32) == cell)
                --j;
            const uint32_t rf = run_of(uint32_t(keys[j]), lines, run, runs_per_view);
            const unsigned long long at = atomicAdd(n, 1ull);
            if (at < cap)
                edges[at] = ((unsigned long long)rf << 32) | (r | kCross);
        }
    }
}

int bits_for(uint64_t v) {
    int b = 1;
    while (b < 64 && (uint64_t(1) << b) <= v)
        ++b;
    return b;
}

// radix sort a[0..n) (bits [0, end_bit)) and drop duplicates; the result is in a
uint64_t sort_unique(unsigned long long* a, unsigned long long* tmp, uint64_t n, int end_bit,
                     unsigned long long* d_num, Scratch& temp, cudaStream_t st) {
    if (n == 0)
        return 0;
    cub::DoubleBuffer<unsigned long long> db(a, tmp);
    size_t tb = 0;
    UB_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, db, int64_t(n), 0, end_bit, st));
    temp.ensure(tb);
    UB_CUDA(cub::DeviceRadixSort::SortKeys(temp.p, tb, db, int64_t(n), 0, end_bit, st));
    unsigned long long* sorted = db.Current();
    unsigned long long* other = db.Alternate();
    size_t tu = 0;
    UB_CUDA(cub::DeviceSelect::Unique(nullptr, tu, sorted, other, d_num, int64_t(n), st));
    temp.ensure(tu);
    UB_CUDA(cub::DeviceSelect::Unique(temp.p, tu, sorted, other, d_num, int64_t(n), st));
    unsigned long long m = 0;
    UB_CUDA(cudaMemcpyAsync(&m, d_num, sizeof(m), cudaMemcpyDeviceToHost, st));
    UB_CUDA(cudaStreamSynchronize(st));
    if (other != a)
        UB_CUDA(cudaMemcpyAsync(a, other, sizeof(unsigned long long) * m, cudaMemcpyDeviceToDevice, st));
    return m;
}

void launch_emit_pairs(const TraceArgs& A, int max_recs, int max_cells, uint64_t units, uint64_t c0, uint64_t c1,
                       unsigned long long* keys, uint64_t cap, unsigned long long* counter, cudaStream_t st) {
    const size_t sm = trace_smem_bytes(kNT, max_recs, max_cells);
    UB_CUDA(cudaFuncSetAttribute(emit_pairs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
    for (uint64_t u0 = 0; u0 < units; u0 += (1u << 30)) {
        const uint32_t n = uint32_t(std::min<uint64_t>(units - u0, 1u << 30));
        emit_pairs_kernel<<<n, kNT, sm, st>>>(A, max_recs, uint32_t(u0), c0, c1, keys, cap, counter);
        count_launch();
    }
    UB_CUDA(cudaGetLastError());
}
}  // namespace

void gpu_schedule_edges(const TraceArgs& A, int views, int max_recs, int max_cells, uint64_t cells,
                        uint64_t visits, uint32_t run, uint32_t runs_per_view,
                        std::vector<unsigned long long>& out_edges, cudaStream_t st) {
    const uint64_t units = uint64_t(views) * uint64_t(A.lines);
    const uint32_t runs = uint32_t(views) * runs_per_view;
    // four buffers of `cap` 8-byte entries (keys, sorted keys, edges, sorted
    // edges) within 60% of the free device memory
    size_t free_b = 0, total_b = 0;
    UB_CUDA(cudaMemGetInfo(&free_b, &total_b));
    const uint64_t cap_max = std::max<uint64_t>(1u << 20, uint64_t(double(free_b) * 0.6) / 32);
    int chunks = int(std::max<uint64_t>(1, (visits + visits / 4 + cap_max - 1) / cap_max));
    Scratch keys, ktmp, edges, etmp, temp, counter;
    counter.ensure(4 * sizeof(unsigned long long));
    unsigned long long* cnt = counter.as<unsigned long long>();
    std::vector<unsigned long long> all;
    while (true) {
        bool overflow = false;
        all.clear();
        const uint64_t cap = std::min<uint64_t>(cap_max, (visits + visits / 4) / uint64_t(chunks) + (1u << 20));
        // at most one edge per visit: a cell's first visit makes no in-sweep
        // edge, its last makes the cross-sweep one
        const uint64_t ecap = cap + (1u << 20);
        keys.ensure(cap * 8);
        ktmp.ensure(cap * 8);
        edges.ensure(ecap * 8);
        etmp.ensure(ecap * 8);
        for (int ch = 0; ch < chunks && !overflow; ++ch) {
            const uint64_t c0 = cells * uint64_t(ch) / uint64_t(chunks);
            const uint64_t c1 = cells * uint64_t(ch + 1) / uint64_t(chunks);
            UB_CUDA(cudaMemsetAsync(cnt, 0, 4 * sizeof(unsigned long long), st));
            launch_emit_pairs(A, max_recs, max_cells, units, c0, c1, keys.as<unsigned long long>(), cap, cnt, st);
            unsigned long long nk = 0;
            UB_CUDA(cudaMemcpyAsync(&nk, cnt, sizeof(nk), cudaMemcpyDeviceToHost, st));
            UB_CUDA(cudaStreamSynchronize(st));
            if (nk > cap) {
                overflow = true;
                break;
            }
            cub::DoubleBuffer<unsigned long long> db(keys.as<unsigned long long>(), ktmp.as<unsigned long long>());
            size_t tb = 0;
            const int kbits = 32 + bits_for(c1 - c0);
            UB_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, db, int64_t(nk), 0, kbits, st));
            temp.ensure(tb);
            UB_CUDA(cub::DeviceRadixSort::SortKeys(temp.p, tb, db, int64_t(nk), 0, kbits, st));
            if (nk > 0) {
                edges_kernel<<<1184, 256, 0, st>>>(db.Current(), nk, uint32_t(A.lines), run, runs_per_view,
                                                   edges.as<unsigned long long>(), ecap, cnt + 1);
                count_launch();
                UB_CUDA(cudaGetLastError());
            }
            unsigned long long ne = 0;
            UB_CUDA(cudaMemcpyAsync(&ne, cnt + 1, sizeof(ne), cudaMemcpyDeviceToHost, st));
            UB_CUDA(cudaStreamSynchronize(st));
            if (ne > ecap) {
                overflow = true;
                break;
            }
            const uint64_t m = sort_unique(edges.as<unsigned long long>(), etmp.as<unsigned long long>(), ne,
                                           32 + bits_for(runs), cnt + 2, temp, st);
            const size_t old = all.size();
            all.resize(old + m);
            UB_CUDA(cudaMemcpyAsync(all.data() + old, edges.p, sizeof(unsigned long long) * m,
                                    cudaMemcpyDeviceToHost, st));
            UB_CUDA(cudaStreamSynchronize(st));
        }
        if (!overflow)
            break;
        chunks *= 2;  // a cell range held more visits than expected: finer ranges
    }
    // global dedup (a run's predecessors can come from several cell ranges)
    const uint64_t n = all.size();
    Scratch acc, atmp;
    acc.ensure(std::max<uint64_t>(n, 1) * 8);
    atmp.ensure(std::max<uint64_t>(n, 1) * 8);
    UB_CUDA(cudaMemcpyAsync(acc.p, all.data(), sizeof(unsigned long long) * n, cudaMemcpyHostToDevice, st));
    const uint64_t m = sort_unique(acc.as<unsigned long long>(), atmp.as<unsigned long long>(), n, 64, cnt + 2,
                                   temp, st);
    out_edges.resize(m);
    UB_CUDA(cudaMemcpyAsync(out_edges.data(), acc.p, sizeof(unsigned long long) * m, cudaMemcpyDeviceToHost, st));
    UB_CUDA(cudaStreamSynchronize(st));
}

}  // namespace ub
