// Internal declarations shared by the uscg_b200 translation units.
//
// Device data layout:
//   ring table   RingRow[n_rings + 1] {count u32, head u32, inv_step f64}, index = ring (1-based)
//   record store SoA: phi_a f64[R], phi_b f64[R], key u32[R]
//                key = ring (bits 0-11) | slice (bits 12-30) | dedup-check flag (bit 31)
//   offsets      u32[lines + 1]
//   thetas       f64[views], norm360 already applied (solver.cpp:116)
//   field        f32 [cell_count][S_pad]  (problem-minor; S_pad = 1 for a single volume)
//   projections  f32 [views*lines][S_pad]
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/uscg_b200.h"

namespace ub {

struct RingRow {
    uint32_t count;
    uint32_t head;
    double inv_step;
};

constexpr uint32_t kRingMask = 0xFFFu;
constexpr uint32_t kSliceShift = 12;
constexpr uint32_t kSliceMask = 0x7FFFFu;
constexpr uint32_t kFlagBit = 0x80000000u;
constexpr int kMaxRings = 4095;
constexpr int kMaxSlices = 0x7FFFF;

struct DevGrid {
    int n_rings;
    int n_slices;  // 1 in 2D
    int volume;
    double ring_spacing;
    double slice_height;
    double radius;  // 0.5 * n * ring_spacing, n = 2 * n_rings (grid.hpp:31)
    double eps;     // 1e-9 * radius (geometry.cpp:29)
    double zoff;    // 0.5 * z_extent (grid.hpp:32-34)
    uint32_t cells_per_slice;
    const RingRow* rings;
};

// Everything a block-level trace needs.
struct TraceArgs {
    const uint32_t* off;
    const double* pa;
    const double* pb;
    const uint32_t* key;
    const RingRow* rings;
    const double* theta;  // per view
    uint32_t cells_per_slice;
    int lines;
};

// ---- launch bookkeeping ------------------------------------------------------
void count_launch(uint64_t n = 1);
void set_error(const std::string& msg);

#define UB_CUDA(expr)                                                                     \
    do {                                                                                  \
        cudaError_t _e = (expr);                                                          \
        if (_e != cudaSuccess)                                                            \
            throw ::ub::CudaError(std::string(#expr) + ": " + cudaGetErrorString(_e));    \
    } while (0)

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct NoDevice : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// ---- device helpers ------------------------------------------------------------

// Tracer::trace_line per-chord rotation (tracer.cpp:160-172): add theta, one
// -360 wrap, scale by inv_step, truncate, clamp to ng-1. The seam test is
// |a - b| <= 180 (tracer.cpp:176). Compiled with --fmad=false so every
// operation rounds exactly as the reference's.
__device__ __forceinline__ void rotate_chord(double pa, double pb, double theta, uint32_t count,
                                             double inv_step, int& lo, int& hi, bool& seam) {
    const int ng = static_cast<int>(count);
    double a = pa + theta;
    if (a >= 360.0)
        a -= 360.0;
    double b = pb + theta;
    if (b >= 360.0)
        b -= 360.0;
    int ga = static_cast<int>(a * inv_step);
    if (ga >= ng)
        ga = ng - 1;
    int gb = static_cast<int>(b * inv_step);
    if (gb >= ng)
        gb = ng - 1;
    lo = ga < gb ? ga : gb;
    hi = ga < gb ? gb : ga;
    seam = !(fabs(a - b) <= 180.0);
}

__device__ __forceinline__ bool range_has(int q, int lo, int hi, bool seam) {
    return seam ? (q >= hi || q <= lo) : (q >= lo && q <= hi);
}

// per-record smem packing: lohi = lo | hi << 12 | seam << 24 ; cnt = count | ng << 16
__device__ __forceinline__ uint32_t pack_lohi(int lo, int hi, bool seam, bool flag) {
    return uint32_t(lo) | (uint32_t(hi) << 12) | (uint32_t(seam) << 24) | (uint32_t(flag) << 25);
}
__device__ __forceinline__ int lohi_lo(uint32_t v) { return int(v & 0xFFFu); }
__device__ __forceinline__ int lohi_hi(uint32_t v) { return int((v >> 12) & 0xFFFu); }
__device__ __forceinline__ bool lohi_seam(uint32_t v) { return (v >> 24) & 1u; }
__device__ __forceinline__ bool lohi_flag(uint32_t v) { return (v >> 25) & 1u; }

// Synchronisation scope of a cooperative trace: the whole block, or a group of
// NT consecutive threads synchronised by named barrier `id` (1..15).
template <int NT>
struct BlockSync {
    static constexpr int kThreads = NT;
    __device__ __forceinline__ int tid() const { return threadIdx.x; }
    __device__ __forceinline__ void sync() const { __syncthreads(); }
    __device__ __forceinline__ bool sync_or(bool p) const { return __syncthreads_or(p) != 0; }
};

template <int NT>
struct GroupSync {
    static constexpr int kThreads = NT;
    int id;
    __device__ __forceinline__ int tid() const { return int(threadIdx.x) % NT; }
    __device__ __forceinline__ void sync() const {
        asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(NT) : "memory");
    }
    __device__ __forceinline__ bool sync_or(bool p) const {
        int r;
        asm volatile(
            "{\n .reg .pred pi, po;\n setp.ne.u32 pi, %1, 0;\n bar.red.or.pred po, %2, %3, pi;\n"
            " selp.u32 %0, 1, 0, po;\n}"
            : "=r"(r)
            : "r"(int(p)), "r"(id), "n"(NT)
            : "memory");
        return r != 0;
    }
};

// A single warp as the sync scope.
struct WarpSync {
    static constexpr int kThreads = 32;
    __device__ __forceinline__ int tid() const { return int(threadIdx.x) & 31; }
    __device__ __forceinline__ void sync() const { __syncwarp(); }
    __device__ __forceinline__ bool sync_or(bool p) const { return __any_sync(0xFFFFFFFFu, p) != 0; }
};

// Exclusive scan of a[0..n) in place over the sync scope; a[n] receives the
// total. s_warp must hold NT/32 words. All threads of the scope must call it.
template <class Sync>
__device__ __forceinline__ void block_exclusive_scan(uint32_t* a, int n, uint32_t* s_warp,
                                                     const Sync& sy) {
    constexpr int NT = Sync::kThreads;
    constexpr int NW = NT / 32;
    const int t = sy.tid();
    const int lane = t & 31, warp = t >> 5;
    const int per = (n + NT - 1) / NT;
    const int beg = min(n, t * per);
    const int end = min(n, beg + per);
    uint32_t sum = 0;
    for (int i = beg; i < end; ++i)
        sum += a[i];
    uint32_t x = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
        if (lane >= o)
            x += y;
    }
    if (lane == 31)
        s_warp[warp] = x;
    sy.sync();
    if (warp == 0) {
        uint32_t w = lane < NW ? s_warp[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, w, o);
            if (lane >= o)
                w += y;
        }
        if (lane < NW)
            s_warp[lane] = w;
    }
    sy.sync();
    uint32_t excl = x - sum + (warp > 0 ? s_warp[warp - 1] : 0u);
    for (int i = beg; i < end; ++i) {
        const uint32_t v = a[i];
        a[i] = excl;
        excl += v;
    }
    if (t == 0)
        a[n] = s_warp[NW - 1];
    sy.sync();
}

struct TraceSmem {
    uint32_t* base;  // max_recs
    uint32_t* lohi;  // max_recs
    uint32_t* cnt;   // max_recs: count | ng << 16
    uint32_t* pos;   // max_recs + 1
    uint32_t* warp;  // NT / 32
    uint32_t* idx;   // max_cells
};

// Number of cells of record i not already covered by an earlier record of the
// same (slice, ring) in this line — the TraceScratch stamp dedup
// (tracer.cpp:181-195) restricted to the only records that can collide.
// Earlier records of the same (slice, ring) as record i, collected with one
// backward scan (up to kMaxPartners; more means "scan per cell"). A line's
// records of one slice are contiguous along the ray (a ray crosses each
// z-slab once), so the scan stops at the start of record i's slice block.
constexpr int kMaxPartners = 4;
struct Partners {
    uint32_t lohi[kMaxPartners];
    int n;         // -1: overflow, use the full scan
    uint32_t slo;  // first cell of record i's slice
};

__device__ __forceinline__ bool same_slice(uint32_t bj, uint32_t slo, uint32_t cps) { return bj - slo < cps; }

__device__ __forceinline__ Partners find_partners(const TraceSmem& S, int i, uint32_t cps) {
    Partners P;
    P.n = 0;
    const uint32_t b = S.base[i];
    P.slo = b - b % cps;
    for (int j = i - 1; j >= 0; --j) {
        const uint32_t bj = S.base[j];
        if (!same_slice(bj, P.slo, cps))
            break;
        if (bj != b)
            continue;
        if (P.n == kMaxPartners) {
            P.n = -1;
            break;
        }
        P.lohi[P.n++] = S.lohi[j];
    }
    return P;
}

__device__ __forceinline__ bool covered(const TraceSmem& S, const Partners& P, int i, int q, uint32_t cps) {
    if (P.n >= 0) {
#pragma unroll
        for (int k = 0; k < kMaxPartners; ++k)
            if (k < P.n && range_has(q, lohi_lo(P.lohi[k]), lohi_hi(P.lohi[k]), lohi_seam(P.lohi[k])))
                return true;
        return false;
    }
    const uint32_t b = S.base[i];
    for (int j = i - 1; j >= 0; --j) {
        const uint32_t bj = S.base[j];
        if (!same_slice(bj, P.slo, cps))
            break;
        if (bj != b)
            continue;
        const uint32_t w = S.lohi[j];
        if (range_has(q, lohi_lo(w), lohi_hi(w), lohi_seam(w)))
            return true;
    }
    return false;
}

__device__ __forceinline__ uint32_t dedup_count(const TraceSmem& S, int i, int ng, uint32_t cps) {
    const uint32_t v = S.lohi[i];
    const int lo = lohi_lo(v), hi = lohi_hi(v);
    const Partners P = find_partners(S, i, cps);
    uint32_t c = 0;
    if (!lohi_seam(v)) {
        for (int q = lo; q <= hi; ++q)
            c += !covered(S, P, i, q, cps);
    } else {
        for (int q = hi; q < ng; ++q)
            c += !covered(S, P, i, q, cps);
        for (int q = 0; q <= lo; ++q)
            c += !covered(S, P, i, q, cps);
    }
    return c;
}

// Trace one (line, theta) with the whole block: fills S.idx[0..n) with the
// deduplicated active cells in the reference emission order (chord order,
// then sector order, tracer.cpp:174-197) and returns n. With expand == false
// only the count is produced. All threads must call it; it ends synchronized.
// Generic form: the sync scope may be a named-barrier group; `rings` may point
// to a shared-memory copy of the ring table. r0/r1 are the line's record range.
// Phase 1 of a trace: rotate every record of the line (trace_chord,
// tracer.cpp:104-142) into S.base / S.lohi / S.cnt (count | ng << 16) / S.pos
// (count); returns whether any record carries the dedup flag (all threads).
template <class Sync>
__device__ bool rotate_records(const TraceArgs& A, uint32_t r0, uint32_t r1, double theta,
                               const TraceSmem& S, const RingRow* rings, const Sync& sy) {
    constexpr int NT = Sync::kThreads;
    constexpr int K = 4;  // records per thread with their loads in flight together
    const int n = int(r1 - r0);
    const int t0 = sy.tid();
    bool any_flag = false;
    for (int i0 = t0; i0 < n; i0 += K * NT) {
        uint32_t key[K];
        double pa[K], pb[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int i = i0 + k * NT;
            if (i < n) {
                key[k] = __ldg(A.key + r0 + i);
                pa[k] = __ldg(A.pa + r0 + i);
                pb[k] = __ldg(A.pb + r0 + i);
            }
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int i = i0 + k * NT;
            if (i >= n)
                break;
            const uint32_t ring = key[k] & kRingMask;
            const uint32_t slice = (key[k] >> kSliceShift) & kSliceMask;
            const bool flag = (key[k] & kFlagBit) != 0;
            const RingRow rr = rings[ring];
            int lo, hi;
            bool seam;
            rotate_chord(pa[k], pb[k], theta, rr.count, rr.inv_step, lo, hi, seam);
            S.base[i] = slice * A.cells_per_slice + rr.head;
            S.lohi[i] = pack_lohi(lo, hi, seam, flag);
            const uint32_t ng = rr.count;
            const uint32_t c = seam ? (ng - uint32_t(hi)) + uint32_t(lo) + 1u : uint32_t(hi - lo) + 1u;
            S.cnt[i] = c | (ng << 16);
            S.pos[i] = c;
            any_flag |= flag;
        }
    }
    return sy.sync_or(any_flag);
}

// count and index sum of one unflagged record's sector range base + [lo..hi]
// (or the seam range hi..ng-1, 0..lo): an arithmetic series
__device__ __forceinline__ void range_count_sum(long long b, int lo, int hi, bool seam, int ng,
                                                unsigned long long& c_acc,
                                                unsigned long long& s_acc) {
    long long c, qs;
    if (!seam) {
        c = hi - lo + 1;
        qs = (static_cast<long long>(lo) + hi) * c / 2;
    } else {
        c = (ng - hi) + lo + 1;
        qs = (static_cast<long long>(hi) + ng - 1) * (ng - hi) / 2 + static_cast<long long>(lo) * (lo + 1) / 2;
    }
    c_acc += static_cast<unsigned long long>(c);
    s_acc += static_cast<unsigned long long>(c * b + qs);
}

template <class Sync>
__device__ int scope_trace(const TraceArgs& A, uint32_t r0, uint32_t r1, double theta,
                           const TraceSmem& S, bool expand, const RingRow* rings, const Sync& sy) {
    constexpr int NT = Sync::kThreads;
    const int n = int(r1 - r0);
    const int t0 = sy.tid();
    if (rotate_records(A, r0, r1, theta, S, rings, sy)) {
        for (int i = t0; i < n; i += NT)
            if (lohi_flag(S.lohi[i]))
                S.pos[i] = dedup_count(S, i, int(S.cnt[i] >> 16), A.cells_per_slice);
        sy.sync();
    }
    block_exclusive_scan(S.pos, n, S.warp, sy);
    const int total = int(S.pos[n]);
    if (!expand)
        return total;
    for (int i = t0; i < n; i += NT) {
        uint32_t p = S.pos[i];
        const uint32_t b = S.base[i];
        const uint32_t v = S.lohi[i];
        const int lo = lohi_lo(v), hi = lohi_hi(v);
        const int ng = int(S.cnt[i] >> 16);
        if (!lohi_flag(v)) {
            if (!lohi_seam(v)) {
                for (int q = lo; q <= hi; ++q)
                    S.idx[p++] = b + uint32_t(q);
            } else {
                for (int q = hi; q < ng; ++q)
                    S.idx[p++] = b + uint32_t(q);
                for (int q = 0; q <= lo; ++q)
                    S.idx[p++] = b + uint32_t(q);
            }
        } else {
            const Partners P = find_partners(S, i, A.cells_per_slice);
            auto emit = [&](int q) {
                if (!covered(S, P, i, q, A.cells_per_slice))
                    S.idx[p++] = b + uint32_t(q);
            };
            if (!lohi_seam(v)) {
                for (int q = lo; q <= hi; ++q)
                    emit(q);
            } else {
                for (int q = hi; q < ng; ++q)
                    emit(q);
                for (int q = 0; q <= lo; ++q)
                    emit(q);
            }
        }
    }
    sy.sync();
    return total;
}

template <int NT>
__device__ int block_trace(const TraceArgs& A, int line, double theta, const TraceSmem& S,
                           bool expand) {
    return scope_trace(A, __ldg(A.off + line), __ldg(A.off + line + 1), theta, S, expand, A.rings,
                       BlockSync<NT>{});
}

// dynamic smem bytes for block_trace
inline size_t trace_smem_bytes(int nt, int max_recs, int max_cells) {
    return sizeof(uint32_t) * (size_t(max_recs) * 4 + 1 + nt / 32 + size_t(max_cells));
}

template <int NT>
__device__ __forceinline__ TraceSmem carve_trace_smem(uint32_t* smem, int max_recs) {
    TraceSmem S;
    S.base = smem;
    S.lohi = S.base + max_recs;
    S.cnt = S.lohi + max_recs;
    S.pos = S.cnt + max_recs;
    S.warp = S.pos + max_recs + 1;
    S.idx = S.warp + NT / 32;
    return S;
}

}  // namespace ub
