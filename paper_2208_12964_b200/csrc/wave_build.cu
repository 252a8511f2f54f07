// The wave executor's inputs (mart_sweep.cu) built on the device from the
// traced lists of every (view, line) (trace_dump, unit order):
//
//  * entries: per traced cell {cell | also in the previous line of the view
//    << 31, position in the next line of the view or 0xFFFF}: a block per
//    line hashes the next line's cells in shared memory;
//  * requirements: per line, the progress each other view must have reached
//    before the line may run. Sorting one (cell, unit) key per traced visit
//    puts each cell's visitors in sweep order: a visit's predecessor is the
//    entry before it (in-sweep), and a cell's first visitor waits for its last
//    one (cross-sweep, previous sweep). A requirement on another view is
//    (that view, its line + 1); per (kind, view, other view) the candidates
//    sorted by line keep only those that raise the maximum of the view's
//    earlier lines (progress counters are monotone and a view's lines become
//    ready in order), and a final sort by (line, kind, other view) gives each
//    line's list in the host builder's order.
//
// The same arrays as the host builder (api.cu build_wave_host,
// USCG_HOST_WAVE=1), checked by tests/test_gpu_parity.py. C2: ~0.85 s on the
// host, tens of milliseconds here.
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <cstdint>
#include <vector>

#include "kernels.h"

namespace ub {

namespace {
constexpr int kNT = 256;
constexpr int kHash = 2048;  // >= 2 x the longest line (wave_supported: at most 768 cells)

template <class T>
struct Buf {
    T* p = nullptr;
    size_t n = 0;
    explicit Buf(size_t count) : n(count) { UB_CUDA(cudaMalloc(&p, sizeof(T) * (count ? count : 1))); }
    ~Buf() {
        if (p)
            cudaFree(p);
    }
    Buf(const Buf&) = delete;
    Buf& operator=(const Buf&) = delete;
};

__global__ void ent_init_kernel(const uint32_t* __restrict__ idx, uint64_t total, uint2* __restrict__ ent) {
    const uint64_t k = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k < total)
        ent[k] = make_uint2(idx[k], 0xFFFFu);
}

// block per unit u (not the last line of its view): cells of line u+1 in a
// shared-memory hash (cell -> position), then u's entries look themselves up
__global__ void __launch_bounds__(kNT) ent_link_kernel(const uint32_t* __restrict__ pos,
                                                       const uint32_t* __restrict__ idx, uint32_t L,
                                                       uint2* __restrict__ ent) {
    __shared__ uint32_t hk[kHash];
    __shared__ uint32_t hv[kHash];
    const uint32_t u = blockIdx.x;
    if (u % L == L - 1)
        return;
    for (int i = threadIdx.x; i < kHash; i += kNT)
        hk[i] = 0xFFFFFFFFu;
    __syncthreads();
    const uint32_t b1 = pos[u + 1], e1 = pos[u + 2];
    for (uint32_t k = b1 + threadIdx.x; k < e1; k += kNT) {
        const uint32_t c = idx[k];
        uint32_t h = (c * 2654435761u) & (kHash - 1);
        while (atomicCAS(&hk[h], 0xFFFFFFFFu, c) != 0xFFFFFFFFu)
            h = (h + 1) & (kHash - 1);
        hv[h] = k - b1;
    }
    __syncthreads();
    const uint32_t b0 = pos[u], e0 = pos[u + 1];
    for (uint32_t k = b0 + threadIdx.x; k < e0; k += kNT) {
        const uint32_t c = idx[k];
        uint32_t h = (c * 2654435761u) & (kHash - 1);
        while (hk[h] != 0xFFFFFFFFu && hk[h] != c)
            h = (h + 1) & (kHash - 1);
        if (hk[h] == c) {
            const uint32_t p = hv[h];
            ent[k].y = p;                       // this entry: its position in the next line
            ent[b1 + p].x = c | 0x80000000u;    // the next line's entry: also in this line
        }
    }
}

// one (cell, unit) key per traced visit: block per unit
__global__ void __launch_bounds__(kNT) visit_keys_kernel(const uint32_t* __restrict__ pos,
                                                         const uint32_t* __restrict__ idx,
                                                         unsigned long long* __restrict__ keys) {
    const uint32_t u = blockIdx.x;
    for (uint32_t k = pos[u] + threadIdx.x; k < pos[u + 1]; k += kNT)
        keys[k] = (uint64_t(idx[k]) << 32) | u;
}

// the last visitor of every cell (the sorted keys' group ends)
__global__ void last_visitor_kernel(const unsigned long long* __restrict__ keys, uint64_t n,
                                    uint32_t* __restrict__ last) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n)
        return;
    const unsigned long long k = keys[i];
    if (i + 1 == n || (keys[i + 1] >> 32) != (k >> 32))
        last[k >> 32] = uint32_t(k);
}

// candidate key: xs << 62 | view << 47 | other view << 32 | line << 16 | need
__device__ __forceinline__ unsigned long long cand_key(uint32_t xs, uint32_t v, uint32_t w, uint32_t line,
                                                       uint32_t need) {
    return (uint64_t(xs) << 62) | (uint64_t(v) << 47) | (uint64_t(w) << 32) | (uint64_t(line) << 16) | need;
}

__global__ void __launch_bounds__(kNT) candidates_kernel(const unsigned long long* __restrict__ keys, uint64_t n,
                                                         const uint32_t* __restrict__ last, uint32_t L,
                                                         unsigned long long* __restrict__ cand,
                                                         unsigned long long* __restrict__ count) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    unsigned long long mine[2];
    int m = 0;
    if (i < n) {
        const unsigned long long k = keys[i];
        const uint32_t c = uint32_t(k >> 32), u = uint32_t(k);
        const uint32_t v = u / L;
        const bool first = i == 0 || (keys[i - 1] >> 32) != c;
        if (!first) {
            const uint32_t w = uint32_t(keys[i - 1]);  // the in-sweep predecessor
            if (w / L != v)
                mine[m++] = cand_key(0, v, w / L, u % L, w % L + 1);
        } else {
            const uint32_t w = last[c];  // the previous sweep's last visitor
            if (w / L != v)
                mine[m++] = cand_key(1, v, w / L, u % L, w % L + 1);
        }
    }
    // warp-aggregated append
    const unsigned lane = threadIdx.x & 31;
    const unsigned has = __ballot_sync(0xFFFFFFFFu, m > 0);
    unsigned long long base = 0;
    if (lane == __ffs(has) - 1 && has)
        base = atomicAdd(count, (unsigned long long)__popc(has));
    base = __shfl_sync(0xFFFFFFFFu, base, has ? __ffs(has) - 1 : 0);
    if (m)
        cand[base + __popc(has & ((1u << lane) - 1))] = mine[0];
}

// Condensing the sorted candidates, in parallel: within a (kind, view, other
// view) group, a line's largest need is its last entry; it is kept when it
// exceeds the largest need of the group's earlier lines (a max-scan by group
// over the line maxima, other entries contributing 0). Survivors as
// (unit << 32 | kind << 31 | other view << 16 | need).
__global__ void line_max_kernel(const unsigned long long* __restrict__ cand, uint64_t n,
                                unsigned long long* __restrict__ group, uint32_t* __restrict__ val) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n)
        return;
    const unsigned long long k = cand[i];
    const bool line_max = i + 1 == n || (cand[i + 1] >> 16) != (k >> 16);
    group[i] = k >> 32;
    val[i] = line_max ? uint32_t(k) & 0xFFFFu : 0u;
}

__global__ void survivors_kernel(const unsigned long long* __restrict__ cand, uint64_t n,
                                 const uint32_t* __restrict__ val, const uint32_t* __restrict__ scan, uint32_t L,
                                 unsigned long long* __restrict__ out, unsigned long long* __restrict__ count) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    bool keep = false;
    unsigned long long o = 0;
    if (i < n && val[i] != 0) {
        const unsigned long long k = cand[i];
        const uint32_t prev = (i > 0 && (cand[i - 1] >> 32) == (k >> 32)) ? scan[i - 1] : 0u;
        const uint32_t need = val[i];
        if (need > prev) {
            const uint32_t xs = uint32_t(k >> 62), v = uint32_t(k >> 47) & 0x7FFFu, w = uint32_t(k >> 32) & 0x7FFFu;
            const uint32_t line = uint32_t(k >> 16) & 0xFFFFu;
            o = (uint64_t(v * L + line) << 32) | (uint64_t(xs) << 31) | (uint64_t(w) << 16) | need;
            keep = true;
        }
    }
    const unsigned lane = threadIdx.x & 31;
    const unsigned has = __ballot_sync(0xFFFFFFFFu, keep);
    unsigned long long base = 0;
    if (has && lane == unsigned(__ffs(has) - 1))
        base = atomicAdd(count, (unsigned long long)__popc(has));
    base = __shfl_sync(0xFFFFFFFFu, base, has ? __ffs(has) - 1 : 0);
    if (keep)
        out[base + __popc(has & ((1u << lane) - 1))] = o;
}

__global__ void deps_kernel(const unsigned long long* __restrict__ sorted, uint64_t n, uint32_t* __restrict__ deps,
                            uint32_t* __restrict__ per_unit) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n)
        return;
    const unsigned long long k = sorted[i];
    const uint32_t u = uint32_t(k >> 32);
    deps[2 * i] = ((uint32_t(k) >> 16) & 0x7FFFu) | (uint32_t(k) & 0x80000000u);
    deps[2 * i + 1] = uint32_t(k) & 0xFFFFu;
    atomicAdd(per_unit + u, 1u);
}

int bits_for(uint64_t x) {
    int b = 1;
    while (b < 64 && (uint64_t(1) << b) <= x)
        ++b;
    return b;
}

void sort_keys(unsigned long long*& a, unsigned long long*& b, uint64_t n, int begin_bit, int end_bit,
               cudaStream_t st) {
    cub::DoubleBuffer<unsigned long long> db(a, b);
    size_t tb = 0;
    UB_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, db, int64_t(n), begin_bit, end_bit, st));
    Buf<char> temp(tb);
    UB_CUDA(cub::DeviceRadixSort::SortKeys(temp.p, tb, db, int64_t(n), begin_bit, end_bit, st));
    a = db.Current();
    b = db.Alternate();
}

unsigned blocks(uint64_t n) { return unsigned((n + kNT - 1) / kNT); }
}  // namespace

// ---------------------------------------------------------------------------
// Entries split by cell index mod `parts` (the clustered wave kernel: CTA r
// of a cluster owns the cells with index % parts == r, so a cell handed from
// one line to the next stays in its CTA). Per line and part: the entries in
// line order, each with its position among the next line's entries of the
// same part.
namespace {
__global__ void __launch_bounds__(kNT) split_count_kernel(const uint32_t* __restrict__ pos,
                                                          const uint2* __restrict__ ent, uint32_t parts,
                                                          uint32_t* __restrict__ cnt) {
    __shared__ uint32_t c[8];
    const uint32_t u = blockIdx.x;
    if (threadIdx.x < parts)
        c[threadIdx.x] = 0;
    __syncthreads();
    for (uint32_t k = pos[u] + threadIdx.x; k < pos[u + 1]; k += kNT)
        atomicAdd(&c[(ent[k].x & 0x7FFFFFFFu) % parts], 1u);
    __syncthreads();
    if (threadIdx.x < parts)
        cnt[size_t(parts) * u + threadIdx.x] = c[threadIdx.x];
}

// a warp per line: each entry's rank among the line's entries of its part
__global__ void split_rank_kernel(const uint32_t* __restrict__ pos, const uint2* __restrict__ ent, uint32_t units,
                                  uint32_t parts, uint16_t* __restrict__ li) {
    const uint32_t u = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const unsigned lane = threadIdx.x & 31;
    if (u >= units)
        return;
    uint32_t base[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (uint32_t k0 = pos[u]; k0 < pos[u + 1]; k0 += 32) {
        const uint32_t k = k0 + lane;
        const bool in = k < pos[u + 1];
        const uint32_t part = in ? (ent[k].x & 0x7FFFFFFFu) % parts : 0u;
        const unsigned below = (1u << lane) - 1u;
        for (uint32_t r = 0; r < parts; ++r) {
            const unsigned m = __ballot_sync(0xFFFFFFFFu, in && part == r);
            if (in && part == r)
                li[k] = uint16_t(base[r] + __popc(m & below));
            base[r] += __popc(m);
        }
    }
}

__global__ void __launch_bounds__(kNT) split_fill_kernel(const uint32_t* __restrict__ pos,
                                                         const uint2* __restrict__ ent,
                                                         const uint16_t* __restrict__ li,
                                                         const uint32_t* __restrict__ spos, uint32_t units,
                                                         uint32_t parts, uint2* __restrict__ out) {
    const uint32_t u = blockIdx.x;
    for (uint32_t k = pos[u] + threadIdx.x; k < pos[u + 1]; k += kNT) {
        const uint2 e = ent[k];
        const uint32_t r = (e.x & 0x7FFFFFFFu) % parts;
        const uint32_t nx = e.y == 0xFFFFu ? 0xFFFFu : uint32_t(li[pos[u + 1] + e.y]);
        out[spos[size_t(r) * (units + 1) + u] + li[k]] = make_uint2(e.x, nx);
    }
}
}  // namespace

uint32_t gpu_wave_split(const uint32_t* pos, const uint2* ent, uint64_t total, uint32_t units, uint32_t parts,
                        uint32_t* spos, uint2* split, cudaStream_t st) {
    if (parts < 1 || parts > 8)
        throw CudaError("gpu_wave_split: 1 to 8 parts");
    Buf<uint32_t> cnt(size_t(parts) * units);
    Buf<uint16_t> li(total);
    if (units) {
        split_count_kernel<<<units, kNT, 0, st>>>(pos, ent, parts, cnt.p);
        split_rank_kernel<<<(units + 7) / 8, 256, 0, st>>>(pos, ent, units, parts, li.p);
        UB_CUDA(cudaGetLastError());
    }
    std::vector<uint32_t> c(size_t(parts) * units), sp(size_t(parts) * (size_t(units) + 1));
    UB_CUDA(cudaMemcpyAsync(c.data(), cnt.p, sizeof(uint32_t) * c.size(), cudaMemcpyDeviceToHost, st));
    UB_CUDA(cudaStreamSynchronize(st));
    uint32_t acc = 0, longest = 0;
    for (uint32_t r = 0; r < parts; ++r)
        for (uint32_t u = 0; u <= units; ++u) {
            sp[size_t(r) * (units + 1) + u] = acc;
            if (u < units) {
                acc += c[size_t(parts) * u + r];
                longest = std::max(longest, c[size_t(parts) * u + r]);
            }
        }
    UB_CUDA(cudaMemcpyAsync(spos, sp.data(), sizeof(uint32_t) * sp.size(), cudaMemcpyHostToDevice, st));
    if (units)
        split_fill_kernel<<<units, kNT, 0, st>>>(pos, ent, li.p, spos, units, parts, split);
    UB_CUDA(cudaGetLastError());
    UB_CUDA(cudaStreamSynchronize(st));
    return longest;
}

bool wave_build_supported(uint32_t lines, uint32_t views, uint64_t cells) {
    return lines < 0xFFFFu && views < 0x8000u && cells < (uint64_t(1) << 31);
}

void gpu_wave_build(const uint32_t* pos, const uint32_t* idx, uint64_t total, uint32_t units, uint32_t L,
                    uint32_t views, uint64_t cells, uint2* ent, std::vector<uint32_t>& dep_off,
                    std::vector<uint32_t>& deps, cudaStream_t st) {
    (void)views;
    // entries
    if (total) {
        ent_init_kernel<<<blocks(total), kNT, 0, st>>>(idx, total, ent);
        ent_link_kernel<<<units, kNT, 0, st>>>(pos, idx, L, ent);
        UB_CUDA(cudaGetLastError());
    }
    // visits sorted by (cell, unit)
    Buf<unsigned long long> k0(total), k1(total);
    unsigned long long *ka = k0.p, *kb = k1.p;
    if (total) {
        visit_keys_kernel<<<units, kNT, 0, st>>>(pos, idx, ka);
        sort_keys(ka, kb, total, 0, 32 + bits_for(cells), st);
    }
    Buf<uint32_t> last(cells);
    Buf<unsigned long long> cand(total), ctmp(total), counts(2);
    UB_CUDA(cudaMemsetAsync(counts.p, 0, sizeof(unsigned long long) * 2, st));
    if (total) {
        last_visitor_kernel<<<blocks(total), kNT, 0, st>>>(ka, total, last.p);
        candidates_kernel<<<blocks(total), kNT, 0, st>>>(ka, total, last.p, L, cand.p, counts.p);
        UB_CUDA(cudaGetLastError());
    }
    unsigned long long nc = 0;
    UB_CUDA(cudaMemcpyAsync(&nc, counts.p, sizeof(nc), cudaMemcpyDeviceToHost, st));
    UB_CUDA(cudaStreamSynchronize(st));
    unsigned long long *ca = cand.p, *cb = ctmp.p;
    if (nc) {
        sort_keys(ca, cb, nc, 0, 63, st);
        Buf<unsigned long long> group(nc);
        Buf<uint32_t> val(nc), scan(nc);
        line_max_kernel<<<blocks(nc), kNT, 0, st>>>(ca, nc, group.p, val.p);
        size_t tb = 0;
        UB_CUDA(cub::DeviceScan::InclusiveScanByKey(nullptr, tb, group.p, val.p, scan.p, cub::Max(), int64_t(nc),
                                                    cuda::std::equal_to<>(), st));
        Buf<char> temp(tb);
        UB_CUDA(cub::DeviceScan::InclusiveScanByKey(temp.p, tb, group.p, val.p, scan.p, cub::Max(), int64_t(nc),
                                                    cuda::std::equal_to<>(), st));
        survivors_kernel<<<blocks(nc), kNT, 0, st>>>(ca, nc, val.p, scan.p, L, cb, counts.p + 1);
        UB_CUDA(cudaGetLastError());
    }
    unsigned long long nd = 0;
    UB_CUDA(cudaMemcpyAsync(&nd, counts.p + 1, sizeof(nd), cudaMemcpyDeviceToHost, st));
    UB_CUDA(cudaStreamSynchronize(st));
    // survivors sorted by (unit, kind, other view): each line's list in order
    unsigned long long *sa = cb, *sb = ca;
    Buf<uint32_t> d_deps(2 * nd), per_unit(units);
    UB_CUDA(cudaMemsetAsync(per_unit.p, 0, sizeof(uint32_t) * units, st));
    if (nd) {
        sort_keys(sa, sb, nd, 16, 32 + bits_for(units), st);
        deps_kernel<<<blocks(nd), kNT, 0, st>>>(sa, nd, d_deps.p, per_unit.p);
        UB_CUDA(cudaGetLastError());
    }
    std::vector<uint32_t> cnt(units);
    deps.resize(2 * nd);
    UB_CUDA(cudaMemcpyAsync(cnt.data(), per_unit.p, sizeof(uint32_t) * units, cudaMemcpyDeviceToHost, st));
    if (nd)
        UB_CUDA(cudaMemcpyAsync(deps.data(), d_deps.p, sizeof(uint32_t) * 2 * nd, cudaMemcpyDeviceToHost, st));
    UB_CUDA(cudaStreamSynchronize(st));
    dep_off.assign(size_t(units) + 1, 0);
    for (uint32_t u = 0; u < units; ++u)
        dep_off[u + 1] = dep_off[u] + cnt[u];
}

}  // namespace ub
