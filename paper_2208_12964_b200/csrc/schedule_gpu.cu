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
// are deduplicated per range and again at the end. The rest of AsapSchedule
// also runs here: CSR predecessor lists and per-run counts (atomics + scans),
// merged successor lists (a stable radix sort by predecessor), the ASAP levels
// (a ticket-ordered dataflow kernel: predecessors precede their successors in
// run order) and the level-sorted order (a stable sort by level). C4's
// 18.9 M runs / 0.9 G edges: 2.2 s (host builder: 157 s).
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <utility>
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
    Scratch() = default;
    Scratch(const Scratch&) = delete;
    Scratch& operator=(const Scratch&) = delete;
    void release() {
        if (p)
            cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    bool try_ensure(size_t b) {  // false (no throw) when the device is out of memory
        if (b <= bytes)
            return true;
        release();
        if (cudaMalloc(&p, b) != cudaSuccess) {
            cudaGetLastError();
            p = nullptr;
            return false;
        }
        bytes = b;
        return true;
    }
    void swap(Scratch& o) {
        std::swap(p, o.p);
        std::swap(bytes, o.bytes);
    }
    void ensure(size_t b) {
        if (b <= bytes)
            return;
        release();
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

// block per (view, line): trace, then append (cell - c0, unit) for cells in
// [c0, c1); one global atomic per block reserves the block's slots
__global__ void __launch_bounds__(kNT) emit_pairs_kernel(TraceArgs A, int max_recs, uint32_t unit0, uint64_t c0,
                                                         uint64_t c1, unsigned long long* __restrict__ keys,
                                                         unsigned long long cap, unsigned long long* __restrict__ n) {
    extern __shared__ uint32_t smem[];
    __shared__ uint32_t s_n;
    __shared__ unsigned long long s_base;
    const TraceSmem S = carve_trace_smem<kNT>(smem, max_recs);
    const uint32_t unit = unit0 + blockIdx.x;
    const int v = int(unit / uint32_t(A.lines)), line = int(unit % uint32_t(A.lines));
    if (threadIdx.x == 0)
        s_n = 0;
    const int cnt = block_trace<kNT>(A, line, A.theta[v], S, true);  // ends with a barrier
    uint32_t mine = 0;
    for (int i = threadIdx.x; i < cnt; i += kNT) {
        const uint64_t c = S.idx[i];
        mine += (c >= c0 && c < c1) ? 1u : 0u;
    }
    const uint32_t off = mine ? atomicAdd(&s_n, mine) : 0u;
    __syncthreads();
    if (threadIdx.x == 0)
        s_base = s_n ? atomicAdd(n, (unsigned long long)s_n) : 0ull;
    __syncthreads();
    unsigned long long at = s_base + off;
    for (int i = threadIdx.x; i < cnt; i += kNT) {
        const uint64_t c = S.idx[i];
        if (c < c0 || c >= c1)
            continue;
        if (at < cap)
            keys[at] = ((c - c0) << 32) | unit;
        ++at;
    }
}

// run of each cell's first visitor (the sorted keys' first entry per cell)
__global__ void first_visitor_kernel(const unsigned long long* __restrict__ keys, unsigned long long nkeys,
                                     uint32_t lines, uint32_t run, uint32_t runs_per_view,
                                     uint32_t* __restrict__ first) {
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < nkeys;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long k = keys[i];
        if (i == 0 || uint32_t(keys[i - 1] >> 32) != uint32_t(k >> 32))
            first[k >> 32] = run_of(uint32_t(k), lines, run, runs_per_view);
    }
}

// edges from the sorted (cell, unit) keys; warp-aggregated slot reservation
__global__ void edges_kernel(const unsigned long long* __restrict__ keys, unsigned long long nkeys, uint32_t lines,
                             uint32_t run, uint32_t runs_per_view, const uint32_t* __restrict__ first,
                             unsigned long long* __restrict__ edges, unsigned long long cap,
                             unsigned long long* __restrict__ n) {
    const int lane = threadIdx.x & 31;
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    // block-uniform trip count: whole warps take part in the scan below
    for (unsigned long long base = blockIdx.x * (unsigned long long)blockDim.x; base < nkeys; base += stride) {
        const unsigned long long i = base + threadIdx.x;
        unsigned long long e0 = 0, e1 = 0;
        int ne = 0;
        if (i < nkeys) {
            const unsigned long long k = keys[i];
            const uint32_t cell = uint32_t(k >> 32);
            const uint32_t r = run_of(uint32_t(k), lines, run, runs_per_view);
            if (i > 0 && uint32_t(keys[i - 1] >> 32) == cell) {
                const uint32_t rp = run_of(uint32_t(keys[i - 1]), lines, run, runs_per_view);
                if (rp != r)
                    e0 = ((unsigned long long)r << 32) | rp, ne = 1;
            }
            if (i + 1 == nkeys || uint32_t(keys[i + 1] >> 32) != cell) {
                // the cell's first visitor waits for this (its last) visitor of the previous sweep
                const unsigned long long x = ((unsigned long long)first[cell] << 32) | (r | kCross);
                if (ne)
                    e1 = x;
                else
                    e0 = x;
                ++ne;
            }
        }
        int incl = ne;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= o)
                incl += y;
        }
        const int total = __shfl_sync(0xFFFFFFFFu, incl, 31);
        unsigned long long wbase = 0;
        if (lane == 31 && total)
            wbase = atomicAdd(n, (unsigned long long)total);
        wbase = __shfl_sync(0xFFFFFFFFu, wbase, 31);
        unsigned long long at = wbase + (incl - ne);
        if (ne > 0 && at < cap)
            edges[at] = e0;
        if (ne > 1 && at + 1 < cap)
            edges[at + 1] = e1;
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


namespace {
constexpr int kLvWarps = 8;

// per-run edge counts: in-sweep preds, cross-sweep preds, successors (all)
__global__ void edge_counts_kernel(const unsigned long long* __restrict__ e, unsigned long long m,
                                   uint32_t* __restrict__ npred, uint32_t* __restrict__ npred_x,
                                   uint32_t* __restrict__ nsucc) {
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < m;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long k = e[i];
        const uint32_t u = uint32_t(k >> 32), w = uint32_t(k);
        atomicAdd((w & kCross) ? npred_x + u : npred + u, 1u);
        atomicAdd(nsucc + (w & ~kCross), 1u);
    }
}

// the in-sweep predecessors of each run in CSR order, and the successor
// sort's (pred, succ) pairs. Edges are sorted by (succ, pred word), so a run's
// in-sweep edges lead its block, preds ascending, and an in-sweep edge's CSR
// slot is its index less the cross-sweep edges of the runs before it (xoff).
__global__ void edge_lists_kernel(const unsigned long long* __restrict__ e, unsigned long long m,
                                  const uint32_t* __restrict__ xoff, uint32_t* __restrict__ preds,
                                  uint32_t* __restrict__ skey, uint32_t* __restrict__ sval) {
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < m;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long k = e[i];
        const uint32_t u = uint32_t(k >> 32), w = uint32_t(k);
        if (!(w & kCross))
            preds[i - xoff[u]] = w;
        skey[i] = w & ~kCross;
        sval[i] = u;
    }
}

__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(uint32_t* p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ASAP level of every run (1 + the max level of its in-sweep predecessors,
// which all precede it in run order): a warp per run, blocks take runs in
// ticket order, so a warp only ever waits on runs of blocks already resident
// or finished (no deadlock whatever the scheduling).
__global__ void __launch_bounds__(kLvWarps * 32) levels_kernel(const uint32_t* __restrict__ pred_off,
                                                                const uint32_t* __restrict__ preds, uint32_t runs,
                                                                uint32_t* level, unsigned* ticket) {
    __shared__ uint32_t s_base;
    if (threadIdx.x == 0)
        s_base = atomicAdd(ticket, 1u) * kLvWarps;
    __syncthreads();
    const uint32_t u = s_base + threadIdx.x / 32;
    if (u >= runs)
        return;
    const int lane = threadIdx.x & 31;
    const uint32_t b = pred_off[u], e = pred_off[u + 1];
    uint32_t lev = 0;
    for (uint32_t k = b + lane; k < e; k += 32) {
        const uint32_t* p = level + preds[k];
        uint32_t l;
        while ((l = ld_relaxed(p)) == 0)
            __nanosleep(32);
        lev = l > lev ? l : lev;
    }
    lev = __reduce_max_sync(0xFFFFFFFFu, lev);
    if (lane == 0)
        st_relaxed(level + u, lev + 1);
}

__global__ void iota_kernel(uint32_t* a, uint32_t n) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        a[i] = i;
}

// level_off from the level-sorted keys (levels 1..L are all populated)
__global__ void level_off_kernel(const uint32_t* __restrict__ sorted, uint32_t n, uint32_t* __restrict__ level_off) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        if (i == 0 || sorted[i] != sorted[i - 1])
            level_off[sorted[i] - 1] = i;
        if (i + 1 == n)
            level_off[sorted[i]] = n;
    }
}

using Clock = std::chrono::steady_clock;
double since(Clock::time_point t0, cudaStream_t st) {
    UB_CUDA(cudaStreamSynchronize(st));
    return std::chrono::duration<double>(Clock::now() - t0).count();
}

// the sorted unique edges into acc (device); returns their count
uint64_t device_edges(const TraceArgs& A, int views, int max_recs, int max_cells, uint64_t cells, uint64_t visits,
                      uint32_t run, uint32_t runs_per_view, Scratch& acc, Scratch& temp, Scratch& counter,
                      cudaStream_t st) {
    const uint64_t units = uint64_t(views) * uint64_t(A.lines);
    const uint32_t runs = uint32_t(views) * runs_per_view;
    // four buffers of `cap` 8-byte entries (keys, sorted keys, edges, sorted
    // edges) within 60% of the free device memory
    size_t free_b = 0, total_b = 0;
    UB_CUDA(cudaMemGetInfo(&free_b, &total_b));
    const uint64_t cap_max = std::max<uint64_t>(1u << 20, uint64_t(double(free_b) * 0.6) / 32);
    int chunks = int(std::max<uint64_t>(1, (visits + visits / 4 + cap_max - 1) / cap_max));
    unsigned long long* cnt = counter.as<unsigned long long>();
    // per-range edges are accumulated on the device, or staged on the host
    // when the device has no room for them
    Scratch dacc;
    uint64_t dn = 0;
    bool on_dev = true;
    std::vector<unsigned long long> all;
    auto append = [&](const unsigned long long* src, uint64_t m) {
        if (on_dev && (dn + m) * 8 > dacc.bytes) {
            Scratch grown;
            if (grown.try_ensure(std::max<uint64_t>(2 * (dn + m), 1u << 20) * 8)) {
                if (dn)
                    UB_CUDA(cudaMemcpyAsync(grown.p, dacc.p, dn * 8, cudaMemcpyDeviceToDevice, st));
                UB_CUDA(cudaStreamSynchronize(st));
                dacc.swap(grown);
            } else {
                on_dev = false;
                all.resize(dn);
                if (dn)
                    UB_CUDA(cudaMemcpyAsync(all.data(), dacc.p, dn * 8, cudaMemcpyDeviceToHost, st));
                UB_CUDA(cudaStreamSynchronize(st));
                dacc.release();
            }
        }
        if (on_dev) {
            UB_CUDA(cudaMemcpyAsync(dacc.as<unsigned long long>() + dn, src, m * 8, cudaMemcpyDeviceToDevice, st));
            dn += m;
        } else {
            const size_t old = all.size();
            all.resize(old + m);
            UB_CUDA(cudaMemcpyAsync(all.data() + old, src, m * 8, cudaMemcpyDeviceToHost, st));
            UB_CUDA(cudaStreamSynchronize(st));
        }
    };
    while (true) {
        Scratch keys, ktmp, edges, etmp, first;
        bool overflow = false;
        all.clear();
        dn = 0;
        on_dev = true;
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
                first.ensure((c1 - c0) * sizeof(uint32_t));
                first_visitor_kernel<<<1184, 256, 0, st>>>(db.Current(), nk, uint32_t(A.lines), run, runs_per_view,
                                                           first.as<uint32_t>());
                count_launch();
                edges_kernel<<<1184, 256, 0, st>>>(db.Current(), nk, uint32_t(A.lines), run, runs_per_view,
                                                   first.as<uint32_t>(), edges.as<unsigned long long>(), ecap,
                                                   cnt + 1);
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
            if (chunks == 1) {  // one cell range: already globally unique
                acc.ensure(std::max<uint64_t>(m, 1) * 8);
                UB_CUDA(cudaMemcpyAsync(acc.p, edges.p, sizeof(unsigned long long) * m, cudaMemcpyDeviceToDevice,
                                        st));
                UB_CUDA(cudaStreamSynchronize(st));
                return m;
            }
            append(edges.as<unsigned long long>(), m);
        }
        if (!overflow)
            break;
        chunks *= 2;  // a cell range held more visits than expected: finer ranges
    }
    // global dedup (a run's predecessors can come from several cell ranges)
    Scratch atmp;
    uint64_t n = dn;
    if (on_dev) {
        acc.swap(dacc);
    } else {
        n = all.size();
        acc.ensure(std::max<uint64_t>(n, 1) * 8);
        UB_CUDA(cudaMemcpyAsync(acc.p, all.data(), sizeof(unsigned long long) * n, cudaMemcpyHostToDevice, st));
    }
    atmp.ensure(std::max<uint64_t>(n, 1) * 8);
    return sort_unique(acc.as<unsigned long long>(), atmp.as<unsigned long long>(), n, 64, cnt + 2, temp, st);
}

void exclusive_scan(const uint32_t* in, uint32_t* out, uint64_t n, Scratch& temp, cudaStream_t st) {
    size_t tb = 0;
    UB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, int64_t(n), st));
    temp.ensure(tb);
    UB_CUDA(cub::DeviceScan::ExclusiveSum(temp.p, tb, in, out, int64_t(n), st));
}
}  // namespace

// record offsets: out[0] = 0, out[i + 1] = in[0] + ... + in[i] (n + 1 entries)
void launch_exclusive_scan_u32(const uint32_t* in, uint32_t* out, int n, cudaStream_t st) {
    UB_CUDA(cudaMemsetAsync(out, 0, sizeof(uint32_t), st));
    if (n <= 0)
        return;
    size_t tb = 0;
    UB_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, in, out + 1, int64_t(n), st));
    Scratch temp;
    temp.ensure(tb);
    UB_CUDA(cub::DeviceScan::InclusiveSum(temp.p, tb, in, out + 1, int64_t(n), st));
    UB_CUDA(cudaStreamSynchronize(st));  // before the temp storage is released
}

void gpu_schedule_build(const TraceArgs& A, int views, int max_recs, int max_cells, uint64_t cells, uint64_t visits,
                        uint32_t run, uint32_t runs_per_view, GpuSchedule& out, cudaStream_t st) {
    const uint32_t runs = uint32_t(views) * runs_per_view;
    Scratch acc, temp, counter;
    counter.ensure(4 * sizeof(unsigned long long));
    auto t0 = Clock::now();
    const uint64_t m = device_edges(A, views, max_recs, max_cells, cells, visits, run, runs_per_view, acc, temp,
                                    counter, st);
    out.seconds[0] = since(t0, st);
    t0 = Clock::now();
    const unsigned long long* e = acc.as<unsigned long long>();
    // ---- CSR lists
    Scratch cnt4;  // [4][runs + 1]: in-sweep preds, cross preds, successors, cross offsets
    const size_t R1 = size_t(runs) + 1;
    cnt4.ensure(4 * R1 * 4);
    uint32_t* npred = cnt4.as<uint32_t>();
    uint32_t* xcnt = npred + R1;
    uint32_t* nsucc = xcnt + R1;
    uint32_t* xoff = nsucc + R1;
    UB_CUDA(cudaMemsetAsync(cnt4.p, 0, cnt4.bytes, st));
    if (m > 0) {
        edge_counts_kernel<<<1184, 256, 0, st>>>(e, m, npred, xcnt, nsucc);
        count_launch();
        UB_CUDA(cudaGetLastError());
    }
    uint32_t* npred_x = out.alloc(GpuSchedule::kNpredX, std::max<uint32_t>(runs, 1));
    UB_CUDA(cudaMemcpyAsync(npred_x, xcnt, sizeof(uint32_t) * std::max<uint32_t>(runs, 1),
                            cudaMemcpyDeviceToDevice, st));
    exclusive_scan(xcnt, xoff, R1, temp, st);
    uint32_t* pred_off = out.alloc(GpuSchedule::kPredOff, size_t(runs) + 1);
    uint32_t* succ_off = out.alloc(GpuSchedule::kSuccOff, size_t(runs) + 1);
    exclusive_scan(npred, pred_off, size_t(runs) + 1, temp, st);
    exclusive_scan(nsucc, succ_off, size_t(runs) + 1, temp, st);
    uint32_t np = 0;
    UB_CUDA(cudaMemcpyAsync(&np, pred_off + runs, sizeof(np), cudaMemcpyDeviceToHost, st));
    UB_CUDA(cudaStreamSynchronize(st));
    out.n_preds = np;
    out.n_succs = m;
    uint32_t* preds = out.alloc(GpuSchedule::kPreds, std::max<uint64_t>(np, 1));
    uint32_t* succs = out.alloc(GpuSchedule::kSuccs, std::max<uint64_t>(m, 1));
    if (m > 0) {
        // successors: stable sort of (pred, succ) by pred keeps each run's
        // successors in edge order, as the host builder appends them
        Scratch pairs;
        pairs.ensure(4 * m * 4);
        uint32_t* k0 = pairs.as<uint32_t>();
        uint32_t* v0 = k0 + m;
        uint32_t* k1 = v0 + m;
        edge_lists_kernel<<<1184, 256, 0, st>>>(e, m, xoff, preds, k0, v0);
        count_launch();
        UB_CUDA(cudaGetLastError());
        cub::DoubleBuffer<uint32_t> dk(k0, k1), dv(v0, succs);
        size_t tb = 0;
        UB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, int64_t(m), 0, bits_for(runs), st));
        temp.ensure(tb);
        UB_CUDA(cub::DeviceRadixSort::SortPairs(temp.p, tb, dk, dv, int64_t(m), 0, bits_for(runs), st));
        if (dv.Current() != succs)
            UB_CUDA(cudaMemcpyAsync(succs, dv.Current(), sizeof(uint32_t) * m, cudaMemcpyDeviceToDevice, st));
    }
    acc.release();
    cnt4.release();
    out.seconds[1] = since(t0, st);
    t0 = Clock::now();
    // ---- ASAP levels
    Scratch lv;  // level, iota, sorted levels
    lv.ensure(3 * size_t(std::max<uint32_t>(runs, 1)) * 4 + 16);
    uint32_t* level = lv.as<uint32_t>();
    uint32_t* iota = level + runs;
    uint32_t* sorted = iota + runs;
    unsigned* ticket = reinterpret_cast<unsigned*>(sorted + runs);
    UB_CUDA(cudaMemsetAsync(level, 0, sizeof(uint32_t) * runs, st));
    UB_CUDA(cudaMemsetAsync(ticket, 0, sizeof(unsigned), st));
    if (runs > 0) {
        levels_kernel<<<(runs + kLvWarps - 1) / kLvWarps, kLvWarps * 32, 0, st>>>(pred_off, preds, runs, level,
                                                                                 ticket);
        count_launch();
        UB_CUDA(cudaGetLastError());
    }
    out.seconds[2] = since(t0, st);
    t0 = Clock::now();
    // ---- level-sorted order (stable: runs ascending within a level)
    uint32_t* order = out.alloc(GpuSchedule::kOrder, std::max<uint32_t>(runs, 1));
    uint32_t L = 0;
    if (runs > 0) {
        unsigned* d_max = ticket;
        size_t tb = 0;
        UB_CUDA(cub::DeviceReduce::Max(nullptr, tb, level, d_max, int64_t(runs), st));
        temp.ensure(tb);
        UB_CUDA(cub::DeviceReduce::Max(temp.p, tb, level, d_max, int64_t(runs), st));
        UB_CUDA(cudaMemcpyAsync(&L, d_max, sizeof(L), cudaMemcpyDeviceToHost, st));
        iota_kernel<<<1184, 256, 0, st>>>(iota, runs);
        count_launch();
        UB_CUDA(cudaStreamSynchronize(st));
        tb = 0;
        UB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, level, sorted, iota, order, int64_t(runs), 0,
                                                bits_for(L), st));
        temp.ensure(tb);
        UB_CUDA(cub::DeviceRadixSort::SortPairs(temp.p, tb, level, sorted, iota, order, int64_t(runs), 0,
                                                bits_for(L), st));
    }
    uint32_t* level_off = out.alloc(GpuSchedule::kLevelOff, size_t(L) + 1);
    UB_CUDA(cudaMemsetAsync(level_off, 0, sizeof(uint32_t) * (size_t(L) + 1), st));
    if (runs > 0) {
        level_off_kernel<<<1184, 256, 0, st>>>(sorted, runs, level_off);
        count_launch();
        UB_CUDA(cudaGetLastError());
    }
    out.level_off.resize(size_t(L) + 1);
    UB_CUDA(cudaMemcpyAsync(out.level_off.data(), level_off, sizeof(uint32_t) * (size_t(L) + 1),
                            cudaMemcpyDeviceToHost, st));
    out.seconds[3] = since(t0, st);
}

}  // namespace ub
