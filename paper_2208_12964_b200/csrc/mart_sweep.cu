// K3 (persistent forms): one launch runs one or more Sp-MART sweeps.
//
// The host-built schedule (schedule.h) groups the lines of a sweep into runs
// of R consecutive lines of a view and orders the runs topologically; for
// every run it lists its predecessors (runs that last wrote one of its cells)
// and, for sweeps run back to back, its cross-sweep predecessors. Any
// execution that runs every run after its predecessors, its lines in order,
// performs on every cell exactly the reference's sequence of updates
// (proj/src/solver.cpp:111-136).
//
// Executors sharing the group-level task code below:
//   * mart_flow_kernel (default): dataflow. Tracer CTAs trace every line once,
//     in topological order, into a bounded slab of index lists. Updater groups
//     take (run, problem-chunk) tasks from an atomic queue, stage the run's
//     index lists in shared memory while the run's predecessors finish (one
//     dependency counter per task, polled by one lane), update the run's lines
//     in order, then count in at the successors with gpu-scope release
//     reductions. No grid barrier, no SC fence. Updater groups are 256-thread
//     groups for problem stacks (float4 over 8 problems per cell) and single
//     warps for one problem (3D volumes), so that small tasks keep the machine
//     busy.
//   * mart_wave_kernel (2D stacks, below): one CTA per (view, problem chunk)
//     task, the view's lines in order inside the CTA, other views ordered by
//     per-view progress counters.
#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>

#include "kernels.h"

namespace ub {

namespace {
// largest dynamic shared-memory size set per (kernel, device)
std::mutex g_attr_mu;
std::map<std::pair<const void*, int>, size_t> g_attr;
size_t attr_smem(const void* fn) {
    int dev = 0;
    UB_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_attr_mu);
    auto it = g_attr.find({fn, dev});
    return it == g_attr.end() ? 0 : it->second;
}
void note_attr_smem(const void* fn, size_t smem) {
    int dev = 0;
    UB_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_attr_mu);
    size_t& v = g_attr[{fn, dev}];
    v = std::max(v, smem);
}

constexpr int CTA = 1024;   // threads per CTA (one CTA per SM)
constexpr int TG = 256;     // tracer group / level-barrier group size
// dataflow CTA size: single-warp updaters (one problem) are shared-memory
// bound at ~18 per SM, so their CTA is smaller and gets ~96 registers a thread
template <int P>
constexpr int flow_cta() {
    return P == 1 ? 640 : CTA;
}

// Per problem-chunk width P: KR scalar cells held per thread (P < 4),
// KV float4 (4-problem) vectors per thread (P >= 4), GU threads per dataflow
// updater group. Wide chunks move a cell's problems as one 64 / 128-byte
// segment per L1 wavefront (the per-SM L1 request pipe is the shared resource
// of the scattered gathers); their groups grow so that a thread still holds
// KV = 6 cells of a line (768 cells per group).
template <int P> struct SweepShape;
template <> struct SweepShape<1> { static constexpr int KR = 16, KV = 0, GU = 32; };
template <> struct SweepShape<2> { static constexpr int KR = 6, KV = 0, GU = 256; };
template <> struct SweepShape<4> { static constexpr int KR = 8, KV = 4, GU = 256; };
template <> struct SweepShape<8> { static constexpr int KR = 16, KV = 6, GU = 256; };
template <> struct SweepShape<16> { static constexpr int KR = 16, KV = 6, GU = 512; };
template <> struct SweepShape<32> { static constexpr int KR = 16, KV = 6, GU = 1024; };

template <int G> struct SyncFor {
    using type = GroupSync<G>;
    __device__ static type make(int g) { return type{1 + g}; }
};
template <> struct SyncFor<32> {
    using type = WarpSync;
    __device__ static type make(int) { return WarpSync{}; }
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
// Release-only and acquire-only fences. fence.acq_rel.gpu is MEMBAR.ALL.GPU +
// CCTL.IVALL (an L1 invalidation the publisher does not need, which costs the
// SM's other warps their cached lists); fence.release.gpu is the MEMBAR
// alone. fence.acquire.gpu is CCTL.IVALL alone: after a relaxed poll has
// observed a released count it completes the acquire without re-reading the
// counter (an acquire load would be one more L2 round trip).
__device__ __forceinline__ void fence_release_gpu() { asm volatile("fence.release.gpu;" ::: "memory"); }
__device__ __forceinline__ void fence_acquire_gpu() { asm volatile("fence.acquire.gpu;" ::: "memory"); }
__device__ __forceinline__ void red_relaxed_add(unsigned* p, unsigned v) {
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// 16-byte global -> shared copy through L2 (LDGSTS), completed by
// cp_async_wait_all of the issuing thread
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
    const unsigned d = unsigned(__cvta_generic_to_shared(smem_dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gmem_src) : "memory");
}
// predicated forms (no divergent branch around the asm)
__device__ __forceinline__ void cp_async16_if(bool p, void* smem_dst, const void* gmem_src) {
    const unsigned d = unsigned(__cvta_generic_to_shared(smem_dst));
    asm volatile(
        "{ .reg .pred q; setp.ne.b32 q, %2, 0; @q cp.async.cg.shared.global [%0], [%1], 16; }" ::"r"(d),
        "l"(gmem_src), "r"(int(p))
        : "memory");
}
__device__ __forceinline__ void st_shared_v4_if(bool p, void* smem_dst, float4 v) {
    const unsigned d = unsigned(__cvta_generic_to_shared(smem_dst));
    asm volatile(
        "{ .reg .pred q; setp.ne.b32 q, %1, 0; @q st.shared.v4.f32 [%0], {%2, %3, %4, %5}; }" ::"r"(d),
        "r"(int(p)), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
        : "memory");
}
__device__ __forceinline__ void st_global_cg_v4_if(bool p, void* gmem_dst, float4 v) {
    asm volatile(
        "{ .reg .pred q; setp.ne.b32 q, %1, 0; @q st.global.cg.v4.f32 [%0], {%2, %3, %4, %5}; }" ::"l"(
            gmem_dst),
        "r"(int(p)), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
        : "memory");
}
// L2 eviction-priority forms (createpolicy): the wave executor keeps the
// field rows resident (evict_last) while its traced lists stream (evict_first)
__device__ __forceinline__ uint64_t l2_policy(int kind) {
    uint64_t pol;
    if (kind == 2)
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    else if (kind == 1)
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    else
        asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void cp_async16_hint_if(bool p, void* smem_dst, const void* gmem_src, uint64_t pol) {
    const unsigned d = unsigned(__cvta_generic_to_shared(smem_dst));
    asm volatile(
        "{ .reg .pred q; setp.ne.b32 q, %2, 0; @q cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %3; }" ::"r"(d),
        "l"(gmem_src), "r"(int(p)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void cp_async8_hint_if(bool p, void* smem_dst, const void* gmem_src, uint64_t pol) {
    const unsigned d = unsigned(__cvta_generic_to_shared(smem_dst));
    asm volatile(
        "{ .reg .pred q; setp.ne.b32 q, %2, 0; @q cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %3; }" ::"r"(d),
        "l"(gmem_src), "r"(int(p)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void st_global_cg_v4_hint_if(bool p, void* gmem_dst, float4 v, uint64_t pol) {
    asm volatile(
        "{ .reg .pred q; setp.ne.b32 q, %1, 0; @q st.global.cg.L2::cache_hint.v4.f32 [%0], {%2, %3, %4, %5}, %6; }" ::"l"(
            gmem_dst),
        "r"(int(p)), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Wait until *p >= target, then acquire. The polls are relaxed: a gpu-scope
// acquire load compiles to LDG + CCTL.IVALL, which invalidates the whole L1
// of the SM (the other warps' cached records and offsets) on every poll. The
// final acquire reads a value at least as recent as the one polled
// (coherence), so it synchronizes with the same release.
__device__ __forceinline__ void spin_until_geq(const unsigned* p, unsigned target) {
    unsigned ns = 16;
    while (ld_relaxed(p) < target) {
        __nanosleep(ns);
        ns = ns < 128 ? ns * 2 : 128;
    }
    fence_acquire_gpu();
}

// Shared-memory words of one group: [trace arrays when tracing] + `lists`
// index lists + reduction scratch + meta + per-line cell counts.
__host__ __device__ inline size_t group_words(int P, int G, bool with_trace, int max_recs,
                                              int max_cells, int lists) {
    size_t w = with_trace ? size_t(max_recs) * 4 + 1 + G / 32 : 0;
    w += size_t(max_cells) * size_t(lists);
    w = (w + 3) & ~size_t(3);  // reduction scratch 16-byte aligned
    w += 2 * size_t(G / 32) * P + 2 * size_t(P) + 4 + ((size_t(lists) + 1) & ~size_t(1));
    return w;
}

__host__ __device__ inline size_t round4(size_t w) { return (w + 3) & ~size_t(3); }

__host__ __device__ inline size_t ring_words(int n_rings) {
    return round4((sizeof(RingRow) / 4) * size_t(n_rings + 1));
}

// Pipelined runs (see pipe_run): a slab entry of line j+1 of a run carries
// kPrevMark when its cell is also crossed by line j, and line j carries, per
// position, the position of its cell in line j+1 (kNoNext: none).
constexpr uint32_t kPrevMark = 0x80000000u;
constexpr uint16_t kNoNext = 0xFFFFu;

__host__ __device__ inline int hash_size(int max_cells) {
    int h = 64;
    while (h < 2 * max_cells)
        h <<= 1;
    return h;
}
__host__ __device__ inline size_t npos_words(int run, int max_cells) {
    return round4((size_t(run) * size_t(max_cells) + 1) / 2);
}
// words beyond group_words: tracer = next positions + cell hash (keys, u16
// positions); updater = next positions + the prefetch buffer [max_cells][P]
__host__ __device__ inline size_t tracer_extra(int run, int max_cells) {
    const int H = hash_size(max_cells);
    return npos_words(run, max_cells) + size_t(H) + round4(size_t(H) / 2);
}
__host__ __device__ inline size_t updater_extra(int P, int run, int max_cells) {
    // + the run's line scalars: m [run][P] f32, p_floor [P] f64, active [P] u32
    return npos_words(run, max_cells) + size_t(max_cells) * size_t(P) +
           round4(size_t(run) * P + 3 * size_t(P));
}

// One thread group's state and task code.
template <int P, int G>
struct GroupWorker {
    static constexpr int KR = SweepShape<P>::KR, NCL = G / P;
    using Sync = typename SyncFor<G>::type;
    const MartArgs& A;
    const RingRow* s_rings;
    TraceSmem tr;
    uint32_t* idx0;  // first index list (tr.idx is pointed at the current line's)
    double* red;     // [G/32][P]
    double* fac;     // [P]
    int* meta;       // [0]: cells, [1]: unit, [2]: chunk, [3]: scratch (task id)
    int* line_n;     // [lists]: cells of each staged line
    uint32_t* ext;   // `extra` words after the standard layout (16-byte aligned)
    Sync sy;
    int t;
    // per-line prefetched scalars (valid in threads t < P)
    float m_next = 0.f;
    double pf_next = 0;
    bool act_next = false;

    // group = -1: the group of this thread (threadIdx.x / G); else that
    // group's shared-memory layout (a helper warp working on a group's lines)
    __device__ GroupWorker(const MartArgs& a, uint32_t* smem, int n_rings, bool with_trace,
                           int lists, size_t extra = 0, int group = -1)
        : A(a), s_rings(reinterpret_cast<const RingRow*>(smem)),
          sy(SyncFor<G>::make(int(threadIdx.x) / G)), t(int(threadIdx.x) % G) {
        const int g = group >= 0 ? group : int(threadIdx.x) / G;
        const size_t std_words = round4(group_words(P, G, with_trace, A.max_recs, A.max_cells, lists));
        uint32_t* gbase = smem + ring_words(n_rings) + size_t(g) * (std_words + extra);
        ext = gbase + std_words;
        uint32_t* p = gbase;
        if (with_trace) {
            tr.base = p;
            tr.lohi = tr.base + A.max_recs;
            tr.cnt = tr.lohi + A.max_recs;
            tr.pos = tr.cnt + A.max_recs;
            tr.warp = tr.pos + A.max_recs + 1;
            p = tr.warp + G / 32;
        } else {
            tr.base = tr.lohi = tr.cnt = tr.pos = tr.warp = nullptr;
        }
        tr.idx = p;
        idx0 = p;
        size_t w = size_t(p - gbase) + size_t(A.max_cells) * size_t(lists);
        w = (w + 3) & ~size_t(3);
        red = reinterpret_cast<double*>(gbase + w);
        fac = red + (G / 32) * P;
        meta = reinterpret_cast<int*>(fac + P);
        line_n = meta + 4;
    }

    __device__ void load_scalars(uint32_t unit, int chunk) {
        if (t < P) {
            const size_t c2 = size_t(chunk) * P + t;
            m_next = __ldcs(A.proj + size_t(unit) * A.Sp + c2);  // read once per sweep
            pf_next = __ldg(A.p_floor + c2);
            act_next = __ldg(A.active + c2) != 0;
        }
    }

    // trace (unit, chunk) into the group's smem and prefetch its scalars
    __device__ void prepare(uint32_t unit, int chunk) {
        const int v = int(unit / uint32_t(A.tr.lines)), line = int(unit % uint32_t(A.tr.lines));
        load_scalars(unit, chunk);
        const int n = scope_trace(A.tr, __ldg(A.tr.off + line), __ldg(A.tr.off + line + 1),
                                  __ldg(A.tr.theta + v), tr, true, s_rings, sy);
        if (t == 0) {
            meta[0] = n;
            meta[1] = int(unit);
            meta[2] = chunk;
        }
        sy.sync();
    }

    // mart_update_line (solver.cpp:36-46) for the problems of this thread
    __device__ double line_factor(double p_bar, int chunk) {
        double factor = 0;  // 0: no update
        const double m = double(m_next);
        if (m != 0 && act_next) {
            const double ratio = m / (p_bar > pf_next ? p_bar : pf_next);
            factor = mart_factor(ratio, A.beta, A.power);
            if (factor <= 0) {
                factor = pf_next;
                atomicAdd(A.clamps + size_t(chunk) * P + t, 1ull);
            }
        }
        return factor;
    }

    // A line's update of one problem as an fp32 multiplier and lower bound:
    // factor 0 (skip / inactive) is {1, 0}, the identity on the positive
    // field. The factor is computed in fp64 (solver.cpp:36-46) and rounded
    // once; the reference's clamp keeps the fp64 field strictly positive
    // (solver.cpp:42-45), and an fp32 product below FLT_MIN would underflow
    // to 0, so it saturates at FLT_MIN instead.
    struct Scale {
        float g, lb;
    };
    __device__ static Scale scale_of(double f) {
        return f == 0 ? Scale{1.f, 0.f} : Scale{float(f), FLT_MIN};
    }
    __device__ static float scale_cell(float v, Scale s) { return fmaxf(v * s.g, s.lb); }
    __device__ static float4 scale4(float4 v, Scale a, Scale b, Scale c, Scale d) {
        return make_float4(scale_cell(v.x, a), scale_cell(v.y, b), scale_cell(v.z, c),
                           scale_cell(v.w, d));
    }

    // gather -> reduce -> factor -> scatter for the prepared line
    __device__ void update(unsigned long long* prof = nullptr) {
        if constexpr (P >= 4) {
            update_vec(prof);
            return;
        }
        const int n = meta[0];
        const int chunk = meta[2];
        // element offsets fit 32 bits (cell_count * S_pad < 2^32 is checked on
        // the host), so no 64-bit address stays live across the gather
        const uint32_t Sp = uint32_t(A.Sp);
        const int p = t % P, cl = t / P;
        const uint32_t col = uint32_t(chunk) * P + uint32_t(p);
        float* __restrict__ f = A.field;
        float x[KR];
#pragma unroll
        for (int i = 0; i < KR; ++i) {
            const int c = cl + i * NCL;
            x[i] = c < n ? __ldcg(f + (tr.idx[c] * Sp + col)) : 0.f;
        }
        double sum = 0;
#pragma unroll
        for (int i = 0; i < KR; ++i)
            sum += double(x[i]);
        for (int c = cl + KR * NCL; c < n; c += 4 * NCL) {
            float y[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int cc = c + j * NCL;
                y[j] = cc < n ? __ldcg(f + (tr.idx[cc] * Sp + col)) : 0.f;
            }
#pragma unroll
            for (int j = 0; j < 4; ++j)
                sum += double(y[j]);
        }
#pragma unroll
        for (int o = P; o < 32; o <<= 1)
            sum += __shfl_xor_sync(0xFFFFFFFFu, sum, o);
        double factor;
        if constexpr (G == 32) {
            // one warp: every lane holds its problem's total after the shuffles
            if (prof && t == 0)
                prof[3] = gtimer();
            factor = __shfl_sync(0xFFFFFFFFu, t < P ? line_factor(sum, chunk) : 0.0, p);
            if (prof && t == 0)
                prof[4] = gtimer();
        } else {
            const int lane = t & 31, warp = t >> 5;
            if (lane < P)
                red[warp * P + lane] = sum;
            sy.sync();
            if (prof && t == 0)
                prof[3] = gtimer();
            if (t < P) {
                double p_bar = 0;
#pragma unroll
                for (int w = 0; w < G / 32; ++w)
                    p_bar += red[w * P + t];
                fac[t] = line_factor(p_bar, chunk);
            }
            sy.sync();
            if (prof && t == 0)
                prof[4] = gtimer();
            factor = fac[p];
        }
        if (factor == 0)
            return;
        const Scale sc = scale_of(factor);
#pragma unroll
        for (int i = 0; i < KR; ++i) {
            const int c = cl + i * NCL;
            if (c < n)
                __stcg(f + (tr.idx[c] * Sp + col), scale_cell(x[i], sc));
        }
        for (int c = cl + KR * NCL; c < n; c += 4 * NCL) {
            float y[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int cc = c + j * NCL;
                y[j] = cc < n ? __ldcg(f + (tr.idx[cc] * Sp + col)) : 0.f;
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int cc = c + j * NCL;
                if (cc < n)
                    __stcg(f + (tr.idx[cc] * Sp + col), scale_cell(y[j], sc));
            }
        }
    }

    // A thread's share of p_bar for its 4 problems: the (at most KV) cells it
    // holds are summed in fp32, then the partials join the fp64 cross-lane and
    // cross-warp sums (the reference sums in fp64, solver.cpp:36-40). KV-term
    // fp32 partials bound the relative error of p_bar by (KV-1) * 2^-24, the
    // size of the fp32 field's own rounding per update.
    template <int K>
    __device__ static void partials(const float4* x, double& s0, double& s1, double& s2, double& s3) {
        float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
        for (int i = 0; i < K; ++i) {
            a0 += x[i].x;
            a1 += x[i].y;
            a2 += x[i].z;
            a3 += x[i].w;
        }
        s0 = a0;
        s1 = a1;
        s2 = a2;
        s3 = a3;
    }

    // Vector form for P >= 4: a thread moves the 4 adjacent problems of one
    // cell as one float4 (16 B, aligned: S_pad and the chunk base are
    // multiples of 4), so a task needs a quarter of the load/store
    // instructions and more cell lanes than the scalar form.
    __device__ void update_vec(unsigned long long* prof) {
        constexpr int V = 4, TPC = P / V, NCLV = G / TPC, KV = SweepShape<P>::KV;
        const int n = meta[0];
        const int chunk = meta[2];
        const uint32_t Sp = uint32_t(A.Sp);
        const int q = t % TPC, cl = t / TPC;
        const uint32_t col = uint32_t(chunk) * P + uint32_t(q) * V;
        float4* __restrict__ f4 = reinterpret_cast<float4*>(A.field);
        float4 x[KV];
#pragma unroll
        for (int i = 0; i < KV; ++i) {
            const int c = cl + i * NCLV;
            x[i] = c < n ? __ldcg(f4 + ((tr.idx[c] * Sp + col) >> 2)) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        double s0, s1, s2, s3;
        partials<KV>(x, s0, s1, s2, s3);
        for (int c = cl + KV * NCLV; c < n; c += 2 * NCLV) {
            const int c2 = c + NCLV;
            const float4 y0 = __ldcg(f4 + ((tr.idx[c] * Sp + col) >> 2));
            const float4 y1 = c2 < n ? __ldcg(f4 + ((tr.idx[c2] * Sp + col) >> 2))
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
            s0 += double(y0.x) + double(y1.x);
            s1 += double(y0.y) + double(y1.y);
            s2 += double(y0.z) + double(y1.z);
            s3 += double(y0.w) + double(y1.w);
        }
#pragma unroll
        for (int o = TPC; o < 32; o <<= 1) {
            s0 += __shfl_xor_sync(0xFFFFFFFFu, s0, o);
            s1 += __shfl_xor_sync(0xFFFFFFFFu, s1, o);
            s2 += __shfl_xor_sync(0xFFFFFFFFu, s2, o);
            s3 += __shfl_xor_sync(0xFFFFFFFFu, s3, o);
        }
        const int lane = t & 31, warp = t >> 5;
        if (lane < TPC) {
            double* r = red + warp * P + q * V;
            r[0] = s0;
            r[1] = s1;
            r[2] = s2;
            r[3] = s3;
        }
        sy.sync();
        if (prof && t == 0)
            prof[3] = gtimer();
        factors_to_smem(chunk);
        sy.sync();
        if (prof && t == 0)
            prof[4] = gtimer();
        Scale g0, g1, g2, g3;
        if (!load_scales(q, g0, g1, g2, g3))
            return;
#pragma unroll
        for (int i = 0; i < KV; ++i) {
            const int c = cl + i * NCLV;
            if (c < n)
                __stcg(f4 + ((tr.idx[c] * Sp + col) >> 2), scale4(x[i], g0, g1, g2, g3));
        }
        for (int c = cl + KV * NCLV; c < n; c += NCLV) {
            float4* p4 = f4 + ((tr.idx[c] * Sp + col) >> 2);
            __stcg(p4, scale4(__ldcg(p4), g0, g1, g2, g3));
        }
    }

    // threads t < P: the line's factor of problem t from the warp partials
    // (fp64, solver.cpp:36-46) as its fp32 Scale in the fac slot
    __device__ void factors_to_smem(int chunk) {
        if (t < P) {
            double p_bar = 0;
#pragma unroll
            for (int w = 0; w < G / 32; ++w)
                p_bar += red[w * P + t];
            const Scale s = scale_of(line_factor(p_bar, chunk));
            reinterpret_cast<float2*>(fac)[t] = make_float2(s.g, s.lb);
        }
    }
    // the Scales of problems 4q..4q+3; false when none of them is updated
    __device__ bool load_scales(int q, Scale& a, Scale& b, Scale& c, Scale& d) const {
        const float4 u = reinterpret_cast<const float4*>(fac)[2 * q];
        const float4 w = reinterpret_cast<const float4*>(fac)[2 * q + 1];
        a = Scale{u.x, u.y};
        b = Scale{u.z, u.w};
        c = Scale{w.x, w.y};
        d = Scale{w.z, w.w};
        return (u.y + u.w + w.y + w.w) != 0.f;  // lb = FLT_MIN marks an update
    }
};

__device__ __forceinline__ void stage_rings(uint32_t* smem, const RingRow* rings, int n_rings) {
    RingRow* s = reinterpret_cast<RingRow*>(smem);
    for (int k = threadIdx.x; k <= n_rings; k += blockDim.x)
        s[k] = rings[k];
}
}  // namespace

// dataflow kernel: the larger of the tracer layout (`tgroups` x 256 threads
// with trace arrays; pipelined: a run's lists, next positions and the cell
// hash) and the updater layout (`groups` groups, `run` lists; pipelined: next
// positions and the prefetch buffer). Group counts are the most that fit in
// `budget` bytes.
struct FlowLayout {
    size_t tracer_words, updater_words;  // per group
    int tgroups, groups;
    size_t bytes;
};

static FlowLayout flow_layout(const MartArgs& a, int n_rings, int GU, bool pipe, size_t budget, int cta,
                              bool lists = false) {
    const int P = a.Sp / a.nchunks;
    FlowLayout L;
    L.tracer_words = round4(group_words(P, TG, true, a.max_recs, a.max_cells, pipe ? a.run : 1)) +
                     (pipe ? tracer_extra(a.run, a.max_cells) : 0);
    L.updater_words = round4(group_words(P, GU, GU == 32 && !lists, a.max_recs, a.max_cells, a.run)) +
                      (pipe ? updater_extra(P, a.run, a.max_cells) : 0);
    const size_t avail = budget / sizeof(uint32_t) - ring_words(n_rings);
    L.groups = int(std::min<size_t>(cta / GU, avail / L.updater_words));
    L.tgroups = int(std::min<size_t>(cta / TG, avail / L.tracer_words));
    if (L.groups < 1 || L.tgroups < 1)
        throw CudaError("mart_flow_kernel: a run's index lists do not fit in shared memory");
    L.bytes = sizeof(uint32_t) *
              (ring_words(n_rings) + std::max(L.tracer_words * size_t(L.tgroups),
                                              L.updater_words * size_t(L.groups)));
    return L;
}

// ============================================================================
// dataflow executor
// ============================================================================

struct FlowArgs {
    MartArgs m;
    const uint32_t* order;     // runs in topological (level) order
    const uint32_t* pred_off;  // by run id: in-sweep predecessors = pred_off[r+1] - pred_off[r]
    const uint32_t* succ_off;  // by run id: in-sweep and cross-sweep successors
    const uint32_t* succs;     // successor run ids
    const uint32_t* npred_x;   // by run id: cross-sweep predecessors
    unsigned* count;           // [runs * nchunks]: predecessors completed, cumulative over sweeps
    unsigned* next;            // updater task queue head (zeroed per launch)
    unsigned epoch;            // global index (1-based) of this launch's first sweep
    int n_sweeps;              // sweeps run back to back by this launch
    int n_runs;                // runs per sweep
    int run;                   // lines per run (divides lines per view)
    int runs_per_view;
    int n_rings;
    FlowSlab slab;             // traced index lists, one slot per line
    int tracer_ctas;
    int upd_groups;            // updater groups per CTA (shared-memory bound)
    int tr_groups;             // tracer groups per tracer CTA
    int pipe;                  // pipelined runs (run tracer marks, pipe_run updaters)
    unsigned long long* prof;  // optional: per task phase stamps (ns)
    // single-warp updaters: every (view, line)'s traced list, built once per
    // geometry (null: trace each line from the record store every sweep)
    const uint32_t* lists;
    const unsigned long long* lpos;  // [units + 1]
};

// line (unit) id of line j of run `run`
__device__ __forceinline__ uint32_t run_line(const FlowArgs& a, uint32_t run, int j) {
    const uint32_t view = run / uint32_t(a.runs_per_view);
    const uint32_t r = run % uint32_t(a.runs_per_view);
    return view * uint32_t(a.m.tr.lines) + r * uint32_t(a.run) + uint32_t(j);
}

// Tracer role: trace every line once, in topological run order, into a ring
// of Q slab slots. A slot is rewritten only after every chunk task of its
// previous occupant has copied it.
template <int P>
__device__ void flow_tracer(const FlowArgs& a, GroupWorker<P, TG>& W) {
    const int nchunks = a.m.nchunks;
    const int Q = a.slab.Q;
    int* s_i = W.meta + 3;
    const long long total = (long long)a.n_runs * a.n_sweeps * a.run;
    while (true) {
        if (W.t == 0)
            *s_i = int(atomicAdd(a.slab.tnext, 1u));
        W.sy.sync();
        const int seq = *s_i;  // ((sweep * n_runs) + order position) * run + j
        if (seq >= total)
            break;
        const int pos = (seq / a.run) % a.n_runs;
        const uint32_t unit = run_line(a, __ldg(a.order + pos), seq % a.run);
        const int v = int(unit / uint32_t(a.m.tr.lines)), line = int(unit % uint32_t(a.m.tr.lines));
        const int n = scope_trace(a.m.tr, __ldg(a.m.tr.off + line), __ldg(a.m.tr.off + line + 1),
                                  __ldg(a.m.tr.theta + v), W.tr, true, W.s_rings, W.sy);
        const int slot = seq % Q;
        const unsigned gen = unsigned(seq / Q);
        if (W.t == 0 && gen > 0)
            spin_until_geq(a.slab.used + slot, gen * unsigned(nchunks));
        W.sy.sync();
        uint32_t* dst = a.slab.data + size_t(slot) * a.slab.slot_words;
        for (int c = W.t; c < n; c += TG)
            __stcg(dst + 1 + c, W.tr.idx[c]);
        if (W.t == 0)
            __stcg(dst, uint32_t(n));
        W.sy.sync();
        if (W.t == 0)
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.slab.ready + slot), "r"(gen + 1)
                         : "memory");
    }
}

// Open-addressing cell -> position hash of one line (shared memory, H a power
// of two >= 2 x the longest line; cells of a line are distinct).
__device__ __forceinline__ uint32_t cell_hash(uint32_t cell, int H) {
    return (cell * 2654435761u) >> (32 - __ffs(H) + 1);
}
__device__ __forceinline__ void hash_insert(uint32_t* key, uint16_t* val, int H, uint32_t cell,
                                            uint16_t pos) {
    uint32_t h = cell_hash(cell, H);
    while (atomicCAS(key + h, 0xFFFFFFFFu, cell) != 0xFFFFFFFFu)
        h = (h + 1) & uint32_t(H - 1);
    val[h] = pos;
}
__device__ __forceinline__ int hash_find(const uint32_t* key, const uint16_t* val, int H,
                                         uint32_t cell) {
    uint32_t h = cell_hash(cell, H);
    while (true) {
        const uint32_t k = key[h];
        if (k == cell)
            return val[h];
        if (k == 0xFFFFFFFFu)
            return -1;
        h = (h + 1) & uint32_t(H - 1);
    }
}

// Tracer role for pipelined runs: a group traces a whole run, links its lines
// (line j+1 entries shared with line j get kPrevMark; line j records where
// each of its cells sits in line j+1), then writes the run's slab slots.
// Slot = [n][idx: max_cells][next positions: u16 x max_cells].
template <int P>
__device__ void flow_tracer_runs(const FlowArgs& a, GroupWorker<P, TG>& W) {
    const int nchunks = a.m.nchunks;
    const int Q = a.slab.Q;
    const int R = a.run, mc = a.m.max_cells;
    const int H = hash_size(mc);
    uint16_t* npos = reinterpret_cast<uint16_t*>(W.ext);
    uint32_t* hkey = W.ext + npos_words(R, mc);
    uint16_t* hval = reinterpret_cast<uint16_t*>(hkey + H);
    int* s_i = W.meta + 3;
    for (int c = W.t; c < H; c += TG)
        hkey[c] = 0xFFFFFFFFu;
    const int total = a.n_runs * a.n_sweeps;
    while (true) {
        if (W.t == 0)
            *s_i = int(atomicAdd(a.slab.tnext, 1u));
        W.sy.sync();
        const int rs = *s_i;  // sweep * n_runs + order position
        if (rs >= total)
            break;
        const uint32_t run = __ldg(a.order + rs % a.n_runs);
        for (int j = 0; j < R; ++j) {
            const uint32_t unit = run_line(a, run, j);
            const int v = int(unit / uint32_t(a.m.tr.lines)), line = int(unit % uint32_t(a.m.tr.lines));
            uint32_t* idx = W.idx0 + size_t(j) * mc;
            W.tr.idx = idx;
            const int n = scope_trace(a.m.tr, __ldg(a.m.tr.off + line), __ldg(a.m.tr.off + line + 1),
                                      __ldg(a.m.tr.theta + v), W.tr, true, W.s_rings, W.sy);
            if (W.t == 0)
                W.line_n[j] = n;
            uint16_t* np = npos + size_t(j) * mc;
            for (int c = W.t; c < n; c += TG)
                np[c] = kNoNext;
            if (j > 0) {
                // hash holds line j-1 (cell -> position)
                uint16_t* prev = npos + size_t(j - 1) * mc;
                for (int c = W.t; c < n; c += TG) {
                    const int p = hash_find(hkey, hval, H, idx[c]);
                    if (p >= 0) {
                        prev[p] = uint16_t(c);
                        idx[c] |= kPrevMark;
                    }
                }
                W.sy.sync();
                for (int c = W.t; c < H; c += TG)
                    hkey[c] = 0xFFFFFFFFu;
                W.sy.sync();
            }
            if (j + 1 < R) {
                for (int c = W.t; c < n; c += TG)
                    hash_insert(hkey, hval, H, idx[c] & ~kPrevMark, uint16_t(c));
                W.sy.sync();
            }
        }
        W.tr.idx = W.idx0;
        // the run's slots: wait until their previous occupants were copied
        const int seq0 = rs * R;
        if (W.t < R) {
            const int seq = seq0 + W.t;
            const unsigned gen = unsigned(seq / Q);
            if (gen > 0)
                spin_until_geq(a.slab.used + seq % Q, gen * unsigned(nchunks));
        }
        W.sy.sync();
        for (int j = 0; j < R; ++j) {
            const int n = W.line_n[j];
            uint32_t* dst = a.slab.data + size_t((seq0 + j) % Q) * a.slab.slot_words;
            const uint32_t* idx = W.idx0 + size_t(j) * mc;
            for (int c = W.t; c < n; c += TG)
                __stcg(dst + 1 + c, idx[c]);
            const uint32_t* np = reinterpret_cast<const uint32_t*>(npos + size_t(j) * mc);
            uint32_t* dnp = dst + 1 + mc;
            if ((mc & 1) == 0) {
                for (int c = W.t; c < (n + 1) / 2; c += TG)
                    __stcg(dnp + c, np[c]);
            } else {
                const uint16_t* s16 = npos + size_t(j) * mc;
                uint16_t* d16 = reinterpret_cast<uint16_t*>(dnp);
                for (int c = W.t; c < n; c += TG)
                    d16[c] = s16[c];
            }
            if (W.t == 0)
                __stcg(dst, uint32_t(n));
        }
        W.sy.sync();
        if (W.t < R) {
            const int seq = seq0 + W.t;
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.slab.ready + seq % Q),
                         "r"(unsigned(seq / Q) + 1)
                         : "memory");
        }
    }
}

// A run's lines with the gathers one line ahead (problem chunks P >= 4, 256-
// thread groups, lines of at most KV x (256 / (P/4)) cells). Thread (cl, q)
// owns buffer slots s = cl + i * NCLV of every line, as float4 q of the chunk.
// While line j is reduced and scaled, the cells of line j+1 that line j does
// not cross are copied into the owner's slots (cp.async; they cannot change
// during the run: every other writer is a predecessor or a successor of the
// run); the cells line j does cross are handed over through shared memory by
// line j itself after it has scaled them (no global store, no reload). Every
// cell therefore sees exactly the sequence of updates of the line-by-line
// form, bit for bit (same reduction order, same factors, same rounding).
template <int P, int G>
__device__ void pipe_run(const FlowArgs& a, GroupWorker<P, G>& W, uint32_t run, int chunk,
                         const uint16_t* npos, float4* buf, unsigned long long* prof) {
    constexpr int V = 4, TPC = P / V, NCLV = G / TPC, KV = SweepShape<P>::KV;
    using GW = GroupWorker<P, G>;
    using Scale = typename GW::Scale;
    const int q = W.t % TPC, cl = W.t / TPC;
    const uint32_t Sp4 = uint32_t(a.m.Sp) / V, col4 = (uint32_t(chunk) * P) / V + uint32_t(q);
    float4* __restrict__ f4 = reinterpret_cast<float4*>(a.m.field);
    const int mc = a.m.max_cells;
    auto issue = [&](int j) {
        const uint32_t* idx = W.idx0 + size_t(j) * mc;
        const int n = W.line_n[j];
#pragma unroll
        for (int i = 0; i < KV; ++i) {
            const int s = cl + i * NCLV;
            const uint32_t e = idx[s < n ? s : 0];
            cp_async16_if(s < n && !(e & kPrevMark), buf + s * TPC + q, f4 + (e & ~kPrevMark) * Sp4 + col4);
        }
        cp_async_commit();
    };
    // the run's scalars, staged with the index lists
    const float* sm = reinterpret_cast<const float*>(W.ext + npos_words(a.run, mc) + size_t(mc) * size_t(P));
    const double* spf = reinterpret_cast<const double*>(sm + a.run * P + (P & 1));
    const uint32_t* sact = reinterpret_cast<const uint32_t*>(spf + P);
    if (W.t < P) {
        W.pf_next = spf[W.t];
        W.act_next = sact[W.t] != 0;
    }
    issue(0);
    for (int j = 0; j < a.run; ++j) {
        if (W.t < P)
            W.m_next = sm[j * P + W.t];
        const int n = W.line_n[j];
        const uint32_t* idx = W.idx0 + size_t(j) * mc;
        const uint16_t* np = npos + size_t(j) * mc;
        cp_async_wait_all();
        float4 x[KV];
#pragma unroll
        for (int i = 0; i < KV; ++i) {
            const int s = cl + i * NCLV;
            x[i] = s < n ? buf[s * TPC + q] : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        double s0, s1, s2, s3;
        GW::template partials<KV>(x, s0, s1, s2, s3);
        // the slots are read (the sums depend on every value) before the
        // next line's copies may land in them
        asm volatile("" ::"d"(s0), "d"(s1), "d"(s2), "d"(s3));
        if (j + 1 < a.run)
            issue(j + 1);
#pragma unroll
        for (int o = TPC; o < 32; o <<= 1) {
            s0 += __shfl_xor_sync(0xFFFFFFFFu, s0, o);
            s1 += __shfl_xor_sync(0xFFFFFFFFu, s1, o);
            s2 += __shfl_xor_sync(0xFFFFFFFFu, s2, o);
            s3 += __shfl_xor_sync(0xFFFFFFFFu, s3, o);
        }
        const int lane = W.t & 31, warp = W.t >> 5;
        if (lane < TPC) {
            double* r = W.red + warp * P + q * V;
            r[0] = s0;
            r[1] = s1;
            r[2] = s2;
            r[3] = s3;
        }
        W.sy.sync();
        if (j == 0 && prof && W.t == 0)
            prof[3] = gtimer();
        W.factors_to_smem(chunk);
        W.sy.sync();
        if (j == 0 && prof && W.t == 0)
            prof[4] = gtimer();
        Scale g0, g1, g2, g3;
        W.load_scales(q, g0, g1, g2, g3);  // identity Scales store unchanged values
#pragma unroll
        for (int i = 0; i < KV; ++i) {
            const int s = cl + i * NCLV;
            const bool in = s < n;
            const float4 r = GW::scale4(x[i], g0, g1, g2, g3);
            const uint16_t nx = np[in ? s : 0];
            const uint32_t e = idx[in ? s : 0] & ~kPrevMark;
            // line j+1 takes shared cells from its buffer slot; the others go home
            st_shared_v4_if(in && nx != kNoNext, buf + int(nx) * TPC + q, r);
            st_global_cg_v4_if(in && nx == kNoNext, f4 + e * Sp4 + col4, r);
        }
        // hand-overs visible; this line's stores ordered before the next
        // line's copies
        W.sy.sync();
    }
}

// Updater role: (run, chunk) tasks in topological order. Stage the run's
// index lists while its predecessors of this chunk finish, update the run's
// lines in order (the chain between them stays inside the group), then count
// in at the run's successors.
__device__ __forceinline__ void prefetch_l2(const void* base, size_t elem, uint32_t r0, uint32_t r1) {
    const uintptr_t b = (reinterpret_cast<uintptr_t>(base) + elem * r0) & ~uintptr_t(15);
    const uintptr_t e = (reinterpret_cast<uintptr_t>(base) + elem * r1 + 15) & ~uintptr_t(15);
    if (e > b)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(b), "r"(uint32_t(e - b)) : "memory");
}

// Single-warp updaters: the next task's first-view records (its trace reads
// them from HBM: the store is larger than L2) prefetched into L2 while this
// task publishes. `nxt` (lane 0) is the claimed next task.
__device__ __forceinline__ void prefetch_next(const FlowArgs& a, unsigned nxt, int per_sweep, int total) {
    nxt = __shfl_sync(0xFFFFFFFFu, nxt, 0);
    if ((threadIdx.x & 31) != 0 || int(nxt) >= total)
        return;
    const uint32_t run = __ldg(a.order + (int(nxt) % per_sweep) / a.m.nchunks);
    const uint32_t unit = run_line(a, run, 0);
    if (a.lists) {  // the next task's traced lists
        const unsigned long long l0 = __ldg(a.lpos + unit), l1 = __ldg(a.lpos + unit + a.run);
        const uintptr_t b = reinterpret_cast<uintptr_t>(a.lists + l0) & ~uintptr_t(15);
        const uintptr_t e = (reinterpret_cast<uintptr_t>(a.lists + l1) + 15) & ~uintptr_t(15);
        if (e > b)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(b), "r"(uint32_t(e - b)) : "memory");
        return;
    }
    const uint32_t line = unit % uint32_t(a.m.tr.lines);
    const uint32_t r0 = __ldg(a.m.tr.off + line), r1 = __ldg(a.m.tr.off + line + a.run);
    prefetch_l2(a.m.tr.key, sizeof(uint32_t), r0, r1);
    prefetch_l2(a.m.tr.pa, sizeof(double), r0, r1);
    prefetch_l2(a.m.tr.pb, sizeof(double), r0, r1);
}

template <int P, int G>
__device__ void flow_updater(const FlowArgs& a, GroupWorker<P, G>& W) {
    const int nchunks = a.m.nchunks;
    const int Q = a.slab.Q;
    const int warp = W.t >> 5, lane = W.t & 31;
    int* s_task = W.meta + 3;
    if (W.t == 0)
        *s_task = int(atomicAdd(a.next, 1u));
    W.sy.sync();
    int task = *s_task;
    unsigned long long* prof = nullptr;
    const int per_sweep = a.n_runs * nchunks;
    const int total = per_sweep * a.n_sweeps;
    while (task < total) {
        if (a.prof) {
            prof = a.prof + 16 * size_t(task);
            if (W.t == 0)
                prof[0] = gtimer();
        }
        const int sweep = task / per_sweep;  // 0-based within this launch
        const int pos = (task % per_sweep) / nchunks;
        const int chunk = task % nchunks;
        const uint32_t run = __ldg(a.order + pos);
        // claim the next task early; its latency overlaps this one
        unsigned nxt = 0;
        if (W.t == 0)
            nxt = atomicAdd(a.next, 1u);
        const int seq0 = (sweep * a.n_runs + pos) * a.run;
        // sweep s (global, 1-based) needs s in-sweep and s-1 cross-sweep
        // rounds of the run's predecessors of this chunk counted in
        const unsigned s = a.epoch + unsigned(sweep);
        const unsigned npred = __ldg(a.pred_off + run + 1) - __ldg(a.pred_off + run);
        const unsigned target = s * npred + (s - 1) * __ldg(a.npred_x + run);
        unsigned* cnt = a.count + size_t(run) * nchunks + chunk;
        // the publishing warp loads the run's first 64 successors now: their
        // latency is hidden behind the task instead of stalling the publish
        constexpr int kPub = G == 32 ? 0 : 1;  // publishing warp
        uint32_t sb = 0, se = 0, succ0 = 0, succ1 = 0;
        if (G == 32) {  // (the larger groups have no registers to spare)
            sb = __ldg(a.succ_off + run);
            se = __ldg(a.succ_off + run + 1);
            if (sb + lane < se)
                succ0 = __ldg(a.succs + sb + lane);
            if (sb + 32 + lane < se)
                succ1 = __ldg(a.succs + sb + 32 + lane);
        }
        auto stage_lists = [&](int ct, int nct) {
            // every line's index list of the run (pipelined: and next
            // positions), from the slab into shared memory (L2 reads: slots
            // are rewritten); four loads in flight per thread
            const int mc = a.m.max_cells;
            for (int j = 0; j < a.run; ++j) {
                const uint32_t* src = a.slab.data + size_t((seq0 + j) % Q) * a.slab.slot_words;
                const int n = int(__ldcg(src));
                uint32_t* dst = W.idx0 + size_t(j) * mc;
                auto copy = [&](const uint32_t* s, uint32_t* d, int m) {
                    int c = ct;
                    for (; c + 3 * nct < m; c += 4 * nct) {
                        const uint32_t v0 = __ldcg(s + c), v1 = __ldcg(s + c + nct),
                                       v2 = __ldcg(s + c + 2 * nct), v3 = __ldcg(s + c + 3 * nct);
                        d[c] = v0;
                        d[c + nct] = v1;
                        d[c + 2 * nct] = v2;
                        d[c + 3 * nct] = v3;
                    }
                    for (; c < m; c += nct)
                        d[c] = __ldcg(s + c);
                };
                copy(src + 1, dst, n);
                if (a.pipe) {
                    uint16_t* np = reinterpret_cast<uint16_t*>(W.ext) + size_t(j) * mc;
                    if ((mc & 1) == 0) {
                        copy(src + 1 + mc, reinterpret_cast<uint32_t*>(np), (n + 1) / 2);
                    } else {
                        const uint16_t* s16 = reinterpret_cast<const uint16_t*>(src + 1 + mc);
                        for (int c = ct; c < n; c += nct)
                            np[c] = __ldcg(s16 + c);
                    }
                }
                if (ct == 0)
                    W.line_n[j] = n;
            }
            if (a.pipe) {
                // the run's measurements and the chunk's floors (inputs: never
                // written by the sweep, so they load before the predecessors end)
                float* sm = reinterpret_cast<float*>(
                    W.ext + npos_words(a.run, mc) + size_t(mc) * size_t(P));
                double* spf = reinterpret_cast<double*>(sm + a.run * P + (P & 1));
                uint32_t* sact = reinterpret_cast<uint32_t*>(spf + P);
                const uint32_t c0 = uint32_t(chunk) * P;
                for (int k = ct; k < a.run * P; k += nct)
                    sm[k] = __ldcs(a.m.proj + size_t(run_line(a, run, k / P)) * a.m.Sp + c0 + k % P);
                for (int k = ct; k < P; k += nct) {
                    spf[k] = __ldg(a.m.p_floor + c0 + k);
                    sact[k] = __ldg(a.m.active + c0 + k);
                }
            }
        };
        if constexpr (G == 32) {
            // one problem: every line is updated once per sweep, so the warp
            // traces its run's lines itself (no slab) while the predecessors
            // finish, then lane 0 waits on them
            (void)stage_lists;
            for (int j = 0; j < a.run && a.lists; ++j) {
                // the line's list, traced once per geometry
                const uint32_t unit = run_line(a, run, j);
                const unsigned long long l0 = __ldg(a.lpos + unit);
                const int n = int(__ldg(a.lpos + unit + 1) - l0);
                if (prof && j == 0) {
                    __syncwarp();
                    if (W.t == 0)
                        prof[9] = gtimer() + 0 * unsigned(n);  // metadata loaded
                }
                uint32_t* dst = W.idx0 + size_t(j) * a.m.max_cells;
                const uint32_t* src = a.lists + l0;
                int c = W.t;
                for (; c + 96 < n; c += 128) {
                    const uint32_t v0 = __ldcs(src + c), v1 = __ldcs(src + c + 32), v2 = __ldcs(src + c + 64),
                                   v3 = __ldcs(src + c + 96);
                    dst[c] = v0;
                    dst[c + 32] = v1;
                    dst[c + 64] = v2;
                    dst[c + 96] = v3;
                }
                for (; c < n; c += 32)
                    dst[c] = __ldcs(src + c);
                if (W.t == 0)
                    W.line_n[j] = n;
            }
            for (int j = 0; j < a.run && !a.lists; ++j) {
                const uint32_t unit = run_line(a, run, j);
                const int v = int(unit / uint32_t(a.m.tr.lines));
                const int line = int(unit % uint32_t(a.m.tr.lines));
                W.tr.idx = W.idx0 + size_t(j) * a.m.max_cells;
                const uint32_t r0 = __ldg(a.m.tr.off + line), r1 = __ldg(a.m.tr.off + line + 1);
                const double theta = __ldg(a.m.tr.theta + v);
                if (prof && j == 0) {
                    __syncwarp();
                    if (W.t == 0)
                        prof[9] = gtimer() + 0 * (r0 + r1 + uint32_t(theta));  // metadata loaded
                }
                const int n = scope_trace(a.m.tr, r0, r1, theta, W.tr, true, W.s_rings, W.sy);
                if (W.t == 0)
                    W.line_n[j] = n;
            }
            if (prof && W.t == 0)
                prof[8] = gtimer();  // traced
            if (W.t == 0 && target)
                spin_until_geq(cnt, target);
            W.sy.sync();
        } else {
            // warp 1 waits on the predecessors while warps 0, 2..7 stage
            constexpr int kCopy = G - 32;
            const GroupSync<kCopy> copy_sync{5 + int(threadIdx.x) / G};
            if (warp == 1) {
                if (lane == 0 && target)
                    spin_until_geq(cnt, target);
                if (prof && lane == 0)
                    prof[15] = gtimer();  // predecessors counted in
            } else {
                if (W.t == 0)
                    for (int j = 0; j < a.run; ++j)
                        spin_until_geq(a.slab.ready + (seq0 + j) % Q, unsigned((seq0 + j) / Q) + 1);
                copy_sync.sync();
                stage_lists(W.t < 32 ? W.t : W.t - 32, kCopy);
                copy_sync.sync();
                if (prof && W.t == 0)
                    prof[7] = gtimer();  // lists staged
            }
            // index lists staged and the predecessors counted in (the acquire
            // orders the gathers after their released stores)
            W.sy.sync();
        }
        if (G != 32 && W.t < a.run)
            red_release_add(a.slab.used + (seq0 + W.t) % Q, 1u);
        if (W.t == 0)
            W.meta[2] = chunk;
        if (prof && W.t == 0)
            prof[1] = prof[2] = gtimer();
        bool piped = false;
        if constexpr (P >= 4 && G >= TG) {
            if (a.pipe) {
                const uint16_t* npos = reinterpret_cast<const uint16_t*>(W.ext);
                float4* buf = reinterpret_cast<float4*>(W.ext + npos_words(a.run, a.m.max_cells));
                pipe_run<P, G>(a, W, run, chunk, npos, buf, prof);
                piped = true;
            }
        }
        if (!piped) {
            for (int j = 0; j < a.run; ++j) {
                // later lines of the run follow the group's own stores (sync below)
                W.load_scalars(run_line(a, run, j), chunk);
                W.tr.idx = W.idx0 + size_t(j) * a.m.max_cells;
                if (W.t == 0)
                    W.meta[0] = W.line_n[j];
                W.sy.sync();
                W.update(j == 0 ? prof : nullptr);
                W.sy.sync();
            }
        }
        W.tr.idx = W.idx0;
        if (prof && W.t == 0)
            prof[5] = gtimer();
        // count in at the run's successors right away (the chain waits on it):
        // one gpu-scope fence (cumulative over the group's stores through the
        // sync above), then a relaxed reduction per successor: fence +
        // relaxed write is a release pattern, with one memory barrier per
        // task instead of one per 32 successors
        {
            if (warp == kPub) {
                if constexpr (G == 32) {
                    fence_release_gpu();
                    if (sb + lane < se)
                        red_relaxed_add(a.count + size_t(succ0) * nchunks + chunk, 1u);
                    if (sb + 32 + lane < se)
                        red_relaxed_add(a.count + size_t(succ1) * nchunks + chunk, 1u);
                    for (uint32_t k = sb + 64 + lane; k < se; k += 32)
                        red_relaxed_add(a.count + size_t(__ldg(a.succs + k)) * nchunks + chunk, 1u);
                    prefetch_next(a, nxt, per_sweep, total);
                } else {
                    sb = __ldg(a.succ_off + run);
                    se = __ldg(a.succ_off + run + 1);
                    fence_release_gpu();
                    for (uint32_t k = sb + lane; k < se; k += 32)
                        red_relaxed_add(a.count + size_t(__ldg(a.succs + k)) * nchunks + chunk, 1u);
                }
                if (prof && lane == 0)
                    prof[6] = gtimer();
            }
        }
        if (W.t == 0)
            *s_task = int(nxt);
        W.sy.sync();
        task = *s_task;
    }
}

// LISTS: single-warp updaters fed by precomputed lists (no trace arrays in
// their shared memory; a compile-time layout, as the traced form's)
template <int P, bool LISTS>
__global__ void __launch_bounds__(flow_cta<P>(), 1) mart_flow_kernel(FlowArgs a) {
    extern __shared__ __align__(16) uint32_t smem[];
    stage_rings(smem, a.m.tr.rings, a.n_rings);
    __syncthreads();
    if (int(blockIdx.x) < a.tracer_ctas) {
        if (int(threadIdx.x) / TG >= a.tr_groups)
            return;  // no shared memory left for this group
        if (a.pipe) {
            GroupWorker<P, TG> W(a.m, smem, a.n_rings, true, a.run, tracer_extra(a.run, a.m.max_cells));
            flow_tracer_runs<P>(a, W);
        } else {
            GroupWorker<P, TG> W(a.m, smem, a.n_rings, true, 1);
            flow_tracer<P>(a, W);
        }
    } else {
        constexpr int GU = SweepShape<P>::GU;
        if (int(threadIdx.x) / GU >= a.upd_groups)
            return;  // no shared memory left for this group
        // single-warp updaters trace their own lines (trace arrays needed)
        // unless the lists are precomputed
        GroupWorker<P, GU> W(a.m, smem, a.n_rings, GU == 32 && !LISTS, a.run,
                             a.pipe ? updater_extra(P, a.run, a.m.max_cells) : 0);
        flow_updater<P, GU>(a, W);
    }
}

template <int P, bool LISTS = false>
static void flow_launch_t(FlowArgs& a, int sms, cudaStream_t st) {
    constexpr int GU = SweepShape<P>::GU;
    int dev = 0, optin = 0;
    UB_CUDA(cudaGetDevice(&dev));
    UB_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    // pipelined runs (USCG_PIPE=1): vector chunks, every line within the
    // register tile, positions in 16 bits. Off by default: on the c2 stack the
    // sweep is bound by the per-SM rate of scattered L1 requests and the
    // dependency chain, not by the gather latency it hides.
    a.pipe = 0;
    if constexpr (P >= 4 && GU >= TG) {
        constexpr int cover = SweepShape<P>::KV * (GU / (P / 4));
        const char* e = std::getenv("USCG_PIPE");
        a.pipe = (e ? std::atoi(e) : 0) != 0 && a.m.max_cells <= cover && a.run > 1;
    }
    constexpr int kCta = flow_cta<P>();
    FlowLayout L = flow_layout(a.m, a.n_rings, GU, a.pipe != 0, size_t(optin) - 1024, kCta, LISTS);
    if (a.pipe && L.groups < std::min(2, kCta / GU)) {  // too little shared memory: plain runs
        a.pipe = 0;
        L = flow_layout(a.m, a.n_rings, GU, false, size_t(optin) - 1024, kCta);
    }
    a.upd_groups = L.groups;
    if (const char* e = std::getenv("USCG_UPD_GROUPS"))  // experiments: fewer groups per SM
        a.upd_groups = std::max(1, std::min(L.groups, std::atoi(e)));
    a.tr_groups = L.tgroups;
    const size_t smem = L.bytes;
    UB_CUDA(cudaFuncSetAttribute(mart_flow_kernel<P, LISTS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(smem)));
    int per_sm = 0;
    UB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mart_flow_kernel<P, LISTS>, kCta, smem));
    if (per_sm < 1)
        throw CudaError("mart_flow_kernel cannot be resident (shared memory too large)");
    const int grid = sms * per_sm;
    // tracer CTAs: trace work ~ lines, update work ~ lines * problems (in
    // 8-problem units; measured balance 2.7 : 4 per unit at 4 tracer groups)
    int k = 0;
    if (GU == 32)
        k = 0;  // single-warp updaters trace their own lines
    else if (const char* e = std::getenv("USCG_TRACER_CTAS"))
        k = std::max(1, std::atoi(e));
    else
        k = std::max(1, int(double(grid) * 2.7 * (4.0 / a.tr_groups) /
                                (2.7 * (4.0 / a.tr_groups) + 4.0 * (a.m.Sp / 8.0)) + 0.5));
    a.tracer_ctas = std::min(k, grid - 1);
    if (const char* e = std::getenv("USCG_FLOW_VERBOSE"); e && std::atoi(e))
        std::fprintf(stderr,
                     "mart_flow_kernel: P=%d run=%d pipe=%d grid=%d tracer_ctas=%d tr_groups=%d "
                     "upd_groups=%d smem=%zu\n",
                     P, a.run, a.pipe, grid, a.tracer_ctas, a.tr_groups, a.upd_groups, smem);
    // every CTA must be resident: tracers and updaters wait on each other
    mart_flow_kernel<P, LISTS><<<grid, kCta, smem, st>>>(a);
}

void launch_mart_flow(const MartArgs& h, const FlowSchedule& fs, unsigned* count, unsigned* next,
                      unsigned epoch, int sweeps, int n_rings, const FlowSlab& slab,
                      cudaStream_t st, unsigned long long* prof, const uint32_t* lists,
                      const unsigned long long* lpos) {
    int dev = 0, sms = 0;
    UB_CUDA(cudaGetDevice(&dev));
    UB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    if (uint64_t(fs.n_runs) * uint64_t(fs.run) * uint64_t(h.nchunks) * uint64_t(sweeps) >= (1ull << 31))
        throw CudaError("mart_flow_kernel: too many tasks for one launch");
    FlowArgs a;
    a.m = h;
    a.order = fs.order;
    a.pred_off = fs.pred_off;
    a.succ_off = fs.succ_off;
    a.succs = fs.succs;
    a.npred_x = fs.npred_x;
    a.count = count;
    a.next = next;
    a.epoch = epoch;
    a.n_sweeps = sweeps;
    a.n_runs = fs.n_runs;
    a.run = fs.run;
    a.runs_per_view = fs.runs_per_view;
    a.n_rings = n_rings;
    a.slab = slab;
    a.tracer_ctas = 1;
    a.prof = prof;
    a.lists = (h.Sp / h.nchunks == 1) ? lists : nullptr;
    a.lpos = a.lists ? lpos : nullptr;
    a.pipe = 0;
    a.tr_groups = CTA / TG;
    a.upd_groups = 1;
    UB_CUDA(cudaMemsetAsync(next, 0, sizeof(unsigned), st));
    UB_CUDA(cudaMemsetAsync(slab.tnext, 0, sizeof(unsigned), st));
    UB_CUDA(cudaMemsetAsync(slab.ready, 0, sizeof(unsigned) * slab.Q, st));
    UB_CUDA(cudaMemsetAsync(slab.used, 0, sizeof(unsigned) * slab.Q, st));
    switch (h.Sp / h.nchunks) {
        case 1: {
            // list-fed single-warp updaters: keep the traced form's layout
            // (trace arrays reserved, unused) when it still fits every group
            // of the CTA — measured faster there (C1 0.92 vs 1.17 ms, C3 5.9
            // vs 6.6 ms per iteration) — else drop the trace arrays to fit
            // more groups (C4: 121 vs 166 ms)
            bool compact = false;
            if (a.lists) {
                int dev = 0, optin = 0;
                UB_CUDA(cudaGetDevice(&dev));
                UB_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
                constexpr int GU = SweepShape<1>::GU, kCta = flow_cta<1>();
                const FlowLayout L = flow_layout(a.m, a.n_rings, GU, false, size_t(optin) - 1024, kCta, false);
                compact = L.groups < kCta / GU;
            }
            if (compact)
                flow_launch_t<1, true>(a, sms, st);
            else
                flow_launch_t<1, false>(a, sms, st);
            break;
        }
        case 2: flow_launch_t<2>(a, sms, st); break;
        case 4: flow_launch_t<4>(a, sms, st); break;
        case 8: flow_launch_t<8>(a, sms, st); break;
        case 16: flow_launch_t<16>(a, sms, st); break;
        case 32: flow_launch_t<32>(a, sms, st); break;
        default: throw CudaError("mart_flow_kernel supports problem chunks of at most 32");
    }
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        throw CudaError(std::string("mart_flow_kernel launch: ") + cudaGetErrorString(e));
}

// ============================================================================
// wave executor (2D problem stacks)
// ============================================================================
//
// A task is one view of one problem chunk in one sweep: a CTA updates the
// view's lines in order, so the chain between consecutive lines of a view
// (adjacent lines of a polar grid always share cells) stays inside the CTA
// and costs a block barrier, not a cross-SM handshake. Lines of other views
// are ordered by one progress counter per (view, chunk), the number of lines
// of that view the chunk has completed (cumulative over sweeps). Every line
// carries the list of other-view counters it needs (the last earlier toucher
// of each of its cells, and for the first toucher of a cell in a sweep, the
// previous sweep's last toucher), condensed on the host to the entries that
// raise a requirement of an earlier line of the view. Executing every line
// after those requirements, the lines of a view in order, performs on every
// cell exactly the reference's sequence of updates (proj/src/solver.cpp:111-136).
//
// CTA = G updater threads (the GroupWorker line code: bit-identical to the
// flow executor's lines) + one control warp. The control warp checks the
// requirements of up to 32 lines per round (one lane per line) and raises
// `ready`; it publishes the updaters' `done` to the view's counter with one
// gpu-scope fence per round (cumulative over the updaters' stores through
// their barrier and the shared-memory release). Tasks are taken in ticket
// order (sweep, view, chunk); a task waits only on smaller tickets, so every
// resident CTA makes progress.

struct WaveArgs {
    MartArgs m;
    const uint32_t* pos;      // [units + 1]: traced list of unit u at ent[pos[u], pos[u+1])
    const uint2* ent;         // per traced entry {cell | in previous line << 31, position in next line}
    const uint32_t* dep_off;  // [units + 1]
    const uint32_t* deps;     // pairs {view | cross-sweep << 31, required line count of that view}
    const uint32_t* spos;     // pair kernel: [2][units + 1] offsets of the entries split by cell parity
    const uint2* split;
    unsigned* prog;           // [views * nchunks] (pair kernel: [views * nchunks][2]): lines completed,
                              // cumulative over sweeps
    unsigned* next;           // task ticket (zeroed per launch)
    unsigned epoch;           // global 0-based index of this launch's first sweep
    int n_sweeps;
    int views;
    int lines;
    unsigned long long* prof;  // optional: per task 8 stamps/sums (ns), see mart_wave_kernel
    int l2_field;              // L2 priority of field rows: 0 normal, 1 evict_first, 2 evict_last
    int l2_lists;              // ... of the traced lists
    unsigned poll_ns;          // requirement poller: longest back-off sleep (ns)
    unsigned pub_ns;           // publisher: sleep between checks of the done count (ns)
};

constexpr uint32_t kWavePrev = 0x80000000u;  // entry's cell is also in the previous line
constexpr uint32_t kWaveNoNext = 0xFFFFu;     // entry's cell is not in the next line
constexpr uint32_t kWavePad = 32;             // one progress counter per 128-byte line (polls of
                                              // neighbouring counters contend in L2)

// Updater shape per chunk width P: G = 16 P threads, TPC = P/4 threads per
// cell (one float4 each), 64 cells per pass and KV = 12 cells per thread (a
// line of up to 768 cells). The CTA is small so that several share an SM:
// one CTA's reduction and barriers overlap another's memory phase (a CTA's
// lines are a dependent chain). MB = CTAs per SM the registers must allow.
// P = 32 (one CTA per SM): 384 threads x 16 cells measured best on C2
// (5.5 ms per iteration; 512 x 12: 5.8, 320 x 20: 5.7, 256 x 24: 5.9).
template <int P> struct WaveShape {
    static constexpr int G = P == 32 ? 384 : 16 * P, KV = P == 32 ? 16 : 12;
    static constexpr int MB = P <= 8 ? 4 : (P == 16 ? 2 : 1);
};
template <int P> __host__ __device__ constexpr int wave_cover() { return WaveShape<P>::KV * (WaveShape<P>::G / (P / 4)); }

__device__ __forceinline__ unsigned ld_acquire_cta_shared(const unsigned* p) {
    unsigned v;
    const unsigned a = unsigned(__cvta_generic_to_shared(p));
    asm volatile("ld.acquire.cta.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_cta_shared(unsigned* p, unsigned v) {
    const unsigned a = unsigned(__cvta_generic_to_shared(p));
    asm volatile("st.release.cta.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_gpu(unsigned* p, unsigned v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void cp_async8_if(bool p, void* smem_dst, const void* gmem_src) {
    const unsigned d = unsigned(__cvta_generic_to_shared(smem_dst));
    asm volatile(
        "{ .reg .pred q; setp.ne.b32 q, %2, 0; @q cp.async.ca.shared.global [%0], [%1], 8; }" ::"r"(d),
        "l"(gmem_src), "r"(int(p))
        : "memory");
}

// dynamic shared memory: [ring words][group words][view offsets L+1]
// [entry ring 3 x cover uint2][field buffer cover x P floats]
template <int P>
__host__ __device__ inline size_t wave_words(int max_recs, int max_cells, int lines) {
    return ring_words(0) + round4(group_words(P, WaveShape<P>::G, false, max_recs, max_cells, 0)) +
           round4(size_t(lines) + 1) + 3 * 2 * size_t(wave_cover<P>()) + size_t(wave_cover<P>()) * P;
}

size_t wave_smem_bytes(const MartArgs& m, int lines) {
    switch (m.Sp / m.nchunks) {
        case 4: return 4 * wave_words<4>(m.max_recs, m.max_cells, lines);
        case 8: return 4 * wave_words<8>(m.max_recs, m.max_cells, lines);
        case 16: return 4 * wave_words<16>(m.max_recs, m.max_cells, lines);
        case 32: return 4 * wave_words<32>(m.max_recs, m.max_cells, lines);
        default: return 0;
    }
}

template <int P>
__global__ void __launch_bounds__(WaveShape<P>::G + 96, WaveShape<P>::MB) mart_wave_kernel(WaveArgs a) {
    constexpr int G = WaveShape<P>::G, V = 4, TPC = P / V, NCLV = G / TPC, KV = WaveShape<P>::KV;
    constexpr int COVER = wave_cover<P>();
    using GW = GroupWorker<P, G>;
    using Scale = typename GW::Scale;
    extern __shared__ __align__(16) uint32_t smem[];
    __shared__ unsigned s_task, s_ready, s_done;
    const int nchunks = a.m.nchunks;
    const unsigned L = unsigned(a.lines);
    const int per_sweep = a.views * nchunks;
    const int total = per_sweep * a.n_sweeps;
    uint32_t* s_pos = smem + ring_words(0) + round4(group_words(P, G, false, a.m.max_recs, a.m.max_cells, 0));
    uint2* s_ent = reinterpret_cast<uint2*>(s_pos + round4(size_t(L) + 1));  // [3][COVER]
    float4* buf = reinterpret_cast<float4*>(s_ent + 3 * COVER);                 // [COVER][TPC]
    if (threadIdx.x == 0) {
        s_task = atomicAdd(a.next, 1u);
        s_ready = 0;
        s_done = 0;
    }
    __syncthreads();
    int task = int(s_task);
    // line barrier (updaters + factor warp) and updater-only barrier
    auto line_sync = [] { asm volatile("bar.sync 1, %0;" ::"n"(G + 32) : "memory"); };
    auto upd_sync = [] { asm volatile("bar.sync 2, %0;" ::"n"(G) : "memory"); };
    if (int(threadIdx.x) >= G && int(threadIdx.x) < G + 32) {
        // ---- factor warp: the line factors (solver.cpp:36-46) from the
        // updaters' partial sums, and the CTA-scope release of `done`. It
        // issues no global stores, so its release fence waits on nothing. ----
        GW W(a.m, smem, 0, false, 0, 0, 0);  // W.t = lane
        const int lane = W.t;
        while (task < total) {
            const int v = (task % per_sweep) / nchunks, chunk = task % nchunks;
            const uint32_t u0 = uint32_t(v) * L;
            float nm = 0.f;
            if (lane < P) {
                const size_t c2 = size_t(chunk) * P + lane;
                W.pf_next = __ldg(a.m.p_floor + c2);
                W.act_next = __ldg(a.m.active + c2) != 0;
                nm = __ldcs(a.m.proj + size_t(u0) * a.m.Sp + c2);
            }
            for (unsigned j = 0; j < L; ++j) {
                W.m_next = nm;
                if (j + 1 < L && lane < P)
                    nm = __ldcs(a.m.proj + size_t(u0 + j + 1) * a.m.Sp + size_t(chunk) * P + lane);
                line_sync();  // A: partial sums in W.red
                W.factors_to_smem(chunk);
                line_sync();  // B: factors in W.fac
                line_sync();  // C: the line's hand-overs and stores issued
                if (lane == 0)
                    st_release_cta_shared(&s_done, j + 1);
            }
            __syncthreads();  // task boundary
            task = int(s_task);
            __syncthreads();
        }
        return;
    }
    if (int(threadIdx.x) >= G + 64) {
        // ---- publisher warp: the lines the updaters have finished (s_done,
        // released by the factor warp after barrier C) become visible at gpu
        // scope: one fence (cumulative over the updaters' stores through the
        // barrier and the shared-memory release) and one relaxed store of the
        // count per round. A warp of its own, so that the fence's wait for the
        // line's stores never delays the requirement polls. ----
        const int lane = int(threadIdx.x) & 31;
        while (task < total) {
            const int sweep = task / per_sweep;
            const int v = (task % per_sweep) / nchunks, chunk = task % nchunks;
            const unsigned gs = a.epoch + unsigned(sweep);
            unsigned* mine = a.prog + (size_t(v) * nchunks + chunk) * kWavePad;
            unsigned long long* lp = a.prof ? a.prof + (8 + 2 * size_t(L)) * size_t(task) + 8 : nullptr;
            unsigned published = 0;
            while (published < L) {
                const unsigned d = ld_acquire_cta_shared(&s_done);
                if (d > published) {
                    if (lane == 0) {
                        fence_release_gpu();
                        st_relaxed_gpu(mine, gs * L + d);
                    }
                    if (lp) {
                        __syncwarp();
                        const unsigned long long tn = gtimer();
                        for (unsigned x = published + unsigned(lane); x < d; x += 32)
                            lp[x] = tn;
                    }
                    published = d;
                } else {
                    __nanosleep(a.pub_ns);
                }
            }
            __syncwarp();
            if (lane == 0) {
                s_task = atomicAdd(a.next, 1u);
                s_ready = 0;
                s_done = 0;
            }
            __syncthreads();  // task boundary (with the updaters)
            task = int(s_task);
            __syncthreads();  // everyone has read the ticket
        }
        return;
    }
    if (int(threadIdx.x) >= G + 32) {
        // ---- poller warp: lane i watches line ready + i. Its requirements
        // (up to kWaveRq counters and counts, the rest re-read from the list)
        // stay in registers, so a poll is one relaxed load per requirement;
        // when lines advance, the lanes shift their cached requirements down
        // by the advance and load the new top lines' ones. An advance is
        // acquired with one gpu-scope fence by the whole warp (every lane that
        // observed a count executes it) and released to the updaters. ----
        constexpr int RQ = 3;
        const int lane = int(threadIdx.x) & 31;
        while (task < total) {
            const int sweep = task / per_sweep;
            const int v = (task % per_sweep) / nchunks, chunk = task % nchunks;
            const unsigned gs = a.epoch + unsigned(sweep);
            unsigned* mine = a.prog + (size_t(v) * nchunks + chunk) * kWavePad;
            const uint32_t u0 = uint32_t(v) * L;
            unsigned long long* lp = a.prof ? a.prof + (8 + 2 * size_t(L)) * size_t(task) + 8 : nullptr;
            // the previous sweep's task of this (view, chunk) has published every line
            if (lane == 0 && gs > 0)
                spin_until_geq(mine, gs * L);
            __syncwarp();
            // cached requirements of line j: n counters (<= RQ here), the rest
            // [kx, ke) of the global list
            uint32_t rc[RQ], rn[RQ];
            int n = 0;
            uint32_t kx = 0, ke = 0;
            auto load_reqs = [&](unsigned j) {
                n = 0;
                kx = ke = 0;
                if (j >= L)
                    return;
                uint32_t k = __ldg(a.dep_off + u0 + j);
                const uint32_t e = __ldg(a.dep_off + u0 + j + 1);
                for (; k < e && n < RQ; ++k) {
                    const uint32_t w = __ldg(a.deps + 2 * size_t(k));
                    const unsigned xs = w >> 31;
                    if (gs < xs)
                        continue;  // no previous sweep
#pragma unroll
                    for (int r = 0; r < RQ; ++r)
                        if (r == n) {
                            rc[r] = ((w & 0x7FFFFFFFu) * unsigned(nchunks) + unsigned(chunk)) * kWavePad;
                            rn[r] = (gs - xs) * L + __ldg(a.deps + 2 * size_t(k) + 1);
                        }
                    ++n;
                }
                kx = k;
                ke = e;
            };
            unsigned ready = 0, ns = 0;
            load_reqs(unsigned(lane));
            while (ready < L) {
                const unsigned j = ready + unsigned(lane);
                bool ok = true;
#pragma unroll
                for (int r = 0; r < RQ; ++r)
                    if (r < n && ok)
                        ok = ld_relaxed(a.prog + rc[r]) >= rn[r];
                for (uint32_t k = kx; k < ke && ok; ++k) {
                    const uint32_t w = __ldg(a.deps + 2 * size_t(k));
                    const unsigned xs = w >> 31;
                    if (gs < xs)
                        continue;
                    const unsigned need = (gs - xs) * L + __ldg(a.deps + 2 * size_t(k) + 1);
                    ok = ld_relaxed(a.prog + (size_t(w & 0x7FFFFFFFu) * nchunks + chunk) * kWavePad) >= need;
                }
                if (j >= L)
                    ok = true;
                const unsigned bad = __ballot_sync(0xFFFFFFFFu, !ok);
                const unsigned adv = bad ? unsigned(__ffs(bad) - 1) : 32u;
                const unsigned nr = min(L, ready + adv);
                if (nr > ready) {
                    // acquire what the advancing lanes observed (an acquire
                    // re-read of a satisfied counter: coherence makes it at
                    // least as recent; a gpu-scope fence here would wait for
                    // the updaters' outstanding stores), then release to the
                    // updaters
                    fence_acquire_gpu();
                    __syncwarp();
                    if (lp) {
                        const unsigned long long tn = gtimer();
                        for (unsigned x = ready + unsigned(lane); x < nr; x += 32)
                            lp[L + x] = tn;
                    }
                    ready = nr;
                    if (lane == 0)
                        st_release_cta_shared(&s_ready, ready);
                    // shift the cached requirements down by adv; new top lines load theirs
                    const int src = lane + int(adv);
#pragma unroll
                    for (int r = 0; r < RQ; ++r) {
                        rc[r] = __shfl_sync(0xFFFFFFFFu, rc[r], src & 31);
                        rn[r] = __shfl_sync(0xFFFFFFFFu, rn[r], src & 31);
                    }
                    n = __shfl_sync(0xFFFFFFFFu, n, src & 31);
                    kx = __shfl_sync(0xFFFFFFFFu, kx, src & 31);
                    ke = __shfl_sync(0xFFFFFFFFu, ke, src & 31);
                    if (src >= 32)
                        load_reqs(ready + unsigned(lane));
                    ns = 0;
                } else {
                    ns = ns ? min(ns * 2, a.poll_ns) : 16u;
                    __nanosleep(ns);
                }
            }
            __syncthreads();  // task boundary (with the updaters)
            task = int(s_task);
            __syncthreads();  // everyone has read the ticket
        }
        return;
    }
    // ---- updaters ----
    // Thread (cl, q) owns slots s = cl + i * NCLV of every line: the entry of
    // the cell at position s (s_ent ring, 2 lines ahead) and float4 q of its
    // problems (buf). A line's cells that the previous line does not cross are
    // copied into the owner's slots during the previous line (cp.async, once
    // the line's requirements hold: no other writer can touch them until this
    // task publishes the line); the cells it does cross are handed over by
    // the previous line after scaling (shared memory; no store, no reload).
    // Every cell sees exactly the line-by-line updates, bit for bit.
    GW W(a.m, smem, 0, false, 0, 0, 0);
    const int t = W.t;
    const int q = t % TPC, cl = t / TPC;
    float4* __restrict__ f4 = reinterpret_cast<float4*>(a.m.field);
    const uint64_t pol_f = l2_policy(a.l2_field), pol_l = l2_policy(a.l2_lists);
    const uint32_t Sp4 = uint32_t(a.m.Sp) / V;
    auto wait_ready = [&](unsigned j) {
        if (ld_acquire_cta_shared(&s_ready) <= j) {
            while (ld_acquire_cta_shared(&s_ready) <= j)
                __nanosleep(16);
        }
    };
    while (task < total) {
        const int v = (task % per_sweep) / nchunks, chunk = task % nchunks;
        const uint32_t u0 = uint32_t(v) * L;
        const uint32_t col4 = (uint32_t(chunk) * P) / V + uint32_t(q);
        for (unsigned j = unsigned(t); j <= L; j += G)
            s_pos[j] = __ldg(a.pos + u0 + j);
        upd_sync();
        // USCG_SWEEP_PROFILE: {start, end, ready-wait, gather, reduce, store} (ns, thread 0)
        const bool prof = a.prof != nullptr && t == 0;
        unsigned long long p_start = prof ? gtimer() : 0, p_wait = 0, p_gather = 0, p_reduce = 0, p_store = 0,
                           p_cwait = 0;
        // entries of line j (own slots) into ring slot j % 3
        auto load_entries = [&](unsigned j) {
            const uint32_t p0 = s_pos[j];
            const int n = int(s_pos[j + 1] - p0);
            uint2* dst = s_ent + (j % 3) * COVER;
#pragma unroll
            for (int i = 0; i < KV; ++i) {
                const int s = cl + i * NCLV;
                cp_async8_hint_if(q == 0 && s < n, dst + s, a.ent + p0 + s, pol_l);
            }
        };
        // field values of line j's cells that line j-1 does not cross (own slots)
        auto gather = [&](unsigned j) {
            const int n = int(s_pos[j + 1] - s_pos[j]);
            const uint2* e = s_ent + (j % 3) * COVER;
#pragma unroll
            for (int i = 0; i < KV; ++i) {
                const int s = cl + i * NCLV;
                const uint32_t c = s < n ? e[s].x : kWavePrev;
                cp_async16_hint_if(!(c & kWavePrev), buf + s * TPC + q, f4 + size_t(c) * Sp4 + col4, pol_f);
            }
        };
        // the entries are written by the slot's q == 0 thread: one barrier
        // makes them visible to the other TPC - 1 threads of the cell
        load_entries(0);
        if (L > 1)
            load_entries(1);
        cp_async_commit();
        cp_async_wait_all();
        upd_sync();
        wait_ready(0);
        gather(0);
        cp_async_commit();
        for (unsigned j = 0; j < L; ++j) {
            const int n = int(s_pos[j + 1] - s_pos[j]);
            const unsigned long long p1 = prof ? gtimer() : 0;
            cp_async_wait_all();  // this line's values (own copies); hand-overs: barrier C
            if (prof)
                p_cwait += gtimer() - p1;
            float4 x[KV];
#pragma unroll
            for (int i = 0; i < KV; ++i) {
                const int s = cl + i * NCLV;
                x[i] = s < n ? buf[s * TPC + q] : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            double s0, s1, s2, s3;
            GW::template partials<KV>(x, s0, s1, s2, s3);
            // the slots are read (the sums depend on every value) before the
            // next line's copies may land in them
            asm volatile("" ::"d"(s0), "d"(s1), "d"(s2), "d"(s3));
#pragma unroll
            for (int o = TPC; o < 32; o <<= 1) {
                s0 += __shfl_xor_sync(0xFFFFFFFFu, s0, o);
                s1 += __shfl_xor_sync(0xFFFFFFFFu, s1, o);
                s2 += __shfl_xor_sync(0xFFFFFFFFu, s2, o);
                s3 += __shfl_xor_sync(0xFFFFFFFFu, s3, o);
            }
            const int lane = t & 31, warp = t >> 5;
            if (lane < TPC) {
                double* r = W.red + warp * P + q * V;
                r[0] = s0;
                r[1] = s1;
                r[2] = s2;
                r[3] = s3;
            }
            line_sync();  // A
            const unsigned long long p2 = prof ? gtimer() : 0;
            // while the factor warp works: entries two lines ahead; the next
            // line's own copies once its requirements hold (its entries,
            // loaded by the cell's q == 0 thread and waited for at this
            // line's start, are visible after barrier A)
            if (j + 2 < L)
                load_entries(j + 2);
            bool issued = false;
            if (j + 1 < L && ld_acquire_cta_shared(&s_ready) > j + 1) {
                gather(j + 1);
                issued = true;
            }
            cp_async_commit();
            line_sync();  // B
            const unsigned long long p3 = prof ? gtimer() : 0;
            Scale g0, g1, g2, g3;
            // identity Scales (none of the thread's 4 problems updated) still
            // hand over, and a cell handed in by the previous line is not in
            // global memory yet: it is stored whatever this line's scales
            const bool any = W.load_scales(q, g0, g1, g2, g3);
            const uint2* e = s_ent + (j % 3) * COVER;
#pragma unroll
            for (int i = 0; i < KV; ++i) {
                const int s = cl + i * NCLV;
                const bool in = s < n;
                const uint2 en = e[in ? s : 0];
                const float4 r = GW::scale4(x[i], g0, g1, g2, g3);
                const bool hand = in && en.y != kWaveNoNext;
                st_shared_v4_if(hand, buf + int(en.y) * TPC + q, r);
                st_global_cg_v4_hint_if((any || (en.x & kWavePrev)) && in && !hand,
                                        f4 + size_t(en.x & ~kWavePrev) * Sp4 + col4, r, pol_f);
            }
            // C: hand-overs visible; this line's stores ordered before the
            // factor warp's release of `done`
            line_sync();
            unsigned long long p4 = prof ? gtimer() : 0, p5 = p4;
            if (!issued && j + 1 < L) {
                wait_ready(j + 1);
                if (prof)
                    p5 = gtimer();
                gather(j + 1);
                cp_async_commit();
            }
            if (prof) {
                p_wait += p5 - p4;
                p_gather += p2 - p1;
                p_reduce += p3 - p2;
                p_store += p4 - p3;
            }
        }
        if (prof) {
            unsigned long long* o = a.prof + (8 + 2 * size_t(L)) * size_t(task);
            o[0] = p_start;
            o[1] = gtimer();
            o[2] = p_wait;
            o[3] = p_gather;
            o[4] = p_reduce;
            o[5] = p_store;
            o[6] = blockIdx.x;
            o[7] = p_cwait;
        }
        __syncthreads();  // task boundary (the control warp grabs the next ticket)
        task = int(s_task);
        __syncthreads();
    }
}

template <int P>
static void wave_launch_t(const WaveArgs& a, int sms, cudaStream_t st) {
    constexpr int NT = WaveShape<P>::G + 96;
    const size_t smem = 4 * wave_words<P>(a.m.max_recs, a.m.max_cells, a.lines);
    // set once per (device, size): changing a running kernel's attributes
    // would wait for it (uscg_reconstruct_batch overlaps neighbouring stacks'
    // solves). The attribute is per device, and contexts on several devices
    // or host threads may launch concurrently.
    if (smem > attr_smem(reinterpret_cast<const void*>(&mart_wave_kernel<P>))) {
        UB_CUDA(cudaFuncSetAttribute(mart_wave_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        note_attr_smem(reinterpret_cast<const void*>(&mart_wave_kernel<P>), smem);
    }
    int per_sm = 0;
    UB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mart_wave_kernel<P>, NT, smem));
    if (per_sm < 1)
        throw CudaError("mart_wave_kernel cannot be resident");
    if (const char* e = std::getenv("USCG_WAVE_PER_SM"))
        per_sm = std::max(1, std::min(per_sm, std::atoi(e)));
    const int total = a.views * a.m.nchunks * a.n_sweeps;
    const int grid = std::min(total, sms * per_sm);
    if (const char* e = std::getenv("USCG_FLOW_VERBOSE"); e && std::atoi(e))
        std::fprintf(stderr, "mart_wave_kernel: P=%d grid=%d per_sm=%d smem=%zu tasks=%d\n", P, grid, per_sm,
                     smem, total);
    // every CTA must be resident: tasks wait on smaller tickets only, held by running CTAs
    mart_wave_kernel<P><<<grid, NT, smem, st>>>(a);
}

// ============================================================================
// wave executor, CTA pairs (P = 32): a view task runs on a 2-CTA cluster
// ============================================================================
//
// The single-CTA wave form spends ~2.4 us of a line's ~2.8 us moving the
// line's rows through one SM's load/store path (profiles/r2_row_microbench.md),
// while the dependency chain leaves SMs idle about half the time. Here the two
// CTAs of a cluster (two SMs) split every line's cells (position s belongs to
// CTA s & 1): each copies, sums, scales, hands over and stores half the rows.
// Per line the partial sums of both CTAs meet through distributed shared
// memory (each factor warp reads both in a fixed order, so both CTAs form the
// same factors), cells handed to the next line go to the owning CTA's buffer
// (st.shared::cluster), and two split mbarriers per CTA (arrivals from the
// updater warps of both CTAs, release/acquire at cluster scope) replace the
// block barriers A and C of the single-CTA form. CTA 0 publishes progress;
// both CTAs' control warps check requirements. Every cell still sees the
// line-by-line updates in order.
namespace pair {
constexpr int V = 4, COVERL = 384;  // cell slots per CTA and task slot
// updater threads per CTA: 384 for 32-problem chunks (8 cells a thread), 256
// for 16 (6 cells a thread); measured on C2: P = 32, 128 problems 4.32 ms
// (256 threads: 4.53, 512: 4.39); P = 16, 16 problems 2.28 ms (384: 2.41)
template <int P> constexpr int updaters() { return P == 16 ? 256 : 384; }
template <int P, int SLOTS> struct Shape {
    static constexpr int GS = updaters<P>() / SLOTS;  // updaters per task slot
    static constexpr int NWS = GS / 32, TPC = P / V, NCLV = GS / TPC, KV = COVERL / NCLV;
    static constexpr int NTS = GS + 96;   // + factor warp + poller warp + publisher warp
    static constexpr int NT = SLOTS * NTS;
};

// dynamic shared memory of one task slot
template <int P, int SLOTS>
__host__ __device__ inline size_t words(int lines) {
    // s_pos | red[NWS][P] f64 | fac[P] float2 | ent[3][COVERL] uint2 | buf[COVERL][P] f32
    return round4(size_t(lines) + 1) + 2 * size_t(Shape<P, SLOTS>::NWS) * P + 2 * size_t(P) +
           3 * 2 * size_t(COVERL) + size_t(COVERL) * P;
}

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t map_peer(const void* p, uint32_t rank) {
    uint32_t d;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(d) : "r"(uint32_t(__cvta_generic_to_shared(p))), "r"(rank));
    return d;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(uint32_t(__cvta_generic_to_shared(b))), "r"(n)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_local(uint64_t* b, unsigned tx) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
                     uint32_t(__cvta_generic_to_shared(b))),
                 "r"(tx)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
    asm volatile(
        "{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(
            uint32_t(__cvta_generic_to_shared(b))),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void st_async_b32(uint32_t cluster_addr, unsigned v, uint32_t cluster_bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(cluster_addr),
                 "r"(v), "r"(cluster_bar)
                 : "memory");
}
__device__ __forceinline__ void st_async_f64(uint32_t cluster_addr, double v, uint32_t cluster_bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(cluster_addr),
                 "l"(__double_as_longlong(v)), "r"(cluster_bar)
                 : "memory");
}
__device__ __forceinline__ void named_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
}  // namespace pair

// CL CTAs per cluster (a view task's cells split by index mod CL), SLOTS
// task slots per CTA (each with its own updaters, factor warp and control
// warp; only SLOTS = 1 is dispatched, see wave_cluster_size).
// At most 112 registers a thread (480 x 112 of the SM's 64 K): uscg_reconstruct_batch
// runs the next stack's small kernels while this one holds every SM, and
// they need the registers left (C2 end to end 5.5 -> 4.5 ms per step; the
// kernel alone 4.10 -> 4.23 ms per iteration at its unconstrained 124).
template <int P, int SLOTS, int CL>
__global__ void __maxnreg__(112) mart_wave_pair_kernel(WaveArgs a) {
    using namespace pair;
    using SH = Shape<P, SLOTS>;
    constexpr int GS = SH::GS, NWS = SH::NWS, TPC = SH::TPC, NCLV = SH::NCLV, KV = SH::KV, NTS = SH::NTS;
    using GW = GroupWorker<P, GS>;
    using Scale = typename GW::Scale;
    extern __shared__ __align__(16) uint32_t smem[];
    __shared__ unsigned s_task[SLOTS], s_ready[SLOTS], s_done[SLOTS];
    __shared__ __align__(8) uint64_t xbar[SLOTS][2], tbar[SLOTS];
    __shared__ __align__(16) double xred[SLOTS][2][CL][P];  // [slot][line parity][CTA][problem]
    const uint32_t rank = cluster_rank();
    const int nchunks = a.m.nchunks;
    const unsigned L = unsigned(a.lines);
    const uint32_t units = uint32_t(a.views) * L;
    const int per_sweep = a.views * nchunks;
    const int total = per_sweep * a.n_sweeps;
    const int tid = int(threadIdx.x);
    const int k = tid / NTS, lt = tid % NTS;  // task slot, thread within the slot
    // this CTA's cells (index % CL == rank): entries split[spos[rank][u] ...]
    const uint32_t* spos = a.spos + size_t(rank) * (units + 1);
    uint32_t* s_pos = smem + size_t(k) * words<P, SLOTS>(int(L));
    double* red = reinterpret_cast<double*>(s_pos + round4(size_t(L) + 1));  // [NWS][P]
    float2* fac = reinterpret_cast<float2*>(red + NWS * P);                  // [P]
    uint2* s_ent = reinterpret_cast<uint2*>(fac + P);                          // [3][COVERL]
    float4* buf = reinterpret_cast<float4*>(s_ent + 3 * COVERL);               // [COVERL][TPC]
    // one progress counter per (view, chunk, CTA): each CTA publishes its own
    // part of a line's cells; a requirement holds when every part does
    auto prog_of = [&](int view, int chunk, uint32_t r) {
        return a.prog + ((size_t(view) * nchunks + chunk) * CL + r) * kWavePad;
    };
    const int id_line = 1 + 3 * k, id_upd = 2 + 3 * k, id_slot = 3 + 3 * k;
    auto line_sync = [&] { named_sync(id_line, GS + 32); };
    auto upd_sync = [&] { named_sync(id_upd, GS); };
    if (lt == 0) {
        mbar_init(&xbar[k][0], 1);
        mbar_init(&xbar[k][1], 1);
        mbar_init(&tbar[k], 1);
        s_ready[k] = 0;
        s_done[k] = 0;
    }
    cluster_sync_all();  // barriers initialised in both CTAs
    // a slot's tasks: CTA 0 takes the ticket and sends it to the peer's slot
    unsigned taken = 0;
    auto next_task = [&](bool first) -> int {
        if (!first)
            named_sync(id_slot, NTS);  // the slot's threads are done with the task
        if (lt == GS + 32) {
            s_ready[k] = 0;
            s_done[k] = 0;
            if (rank == 0) {
                const unsigned t = atomicAdd(a.next, 1u);
                s_task[k] = t;
                for (uint32_t r = 1; r < uint32_t(CL); ++r)
                    st_async_b32(map_peer(&s_task[k], r), t, map_peer(&tbar[k], r));
            } else {
                mbar_arrive_expect_local(&tbar[k], 4);
                mbar_wait(&tbar[k], taken & 1);
            }
        }
        ++taken;
        named_sync(id_slot, NTS);
        return int(s_task[k]);
    };
    int task = next_task(true);
    if (lt >= GS && lt < GS + 32) {
        // ---- factor warp: this CTA's partial sums, exchanged with the peer's
        // slot (st.async into its xred, completing its xbar), both added in
        // the same order in both CTAs (CTA 0's first), then the line factors
        // (solver.cpp:36-46); releases `done` after barrier C ----
        const int lane = lt & 31;
        const bool mine_lane = lane < P;  // lane l: problem l of the chunk
        unsigned jl = 0;
        while (task < total) {
            const int v = (task % per_sweep) / nchunks, chunk = task % nchunks;
            const uint32_t u0 = uint32_t(v) * L;
            const size_t c2 = size_t(chunk) * P + (mine_lane ? lane : 0);
            const double pf = __ldg(a.m.p_floor + c2);
            const bool act = mine_lane && __ldg(a.m.active + c2) != 0;
            float nm = __ldcs(a.m.proj + size_t(u0) * a.m.Sp + c2);
            for (unsigned j = 0; j < L; ++j, ++jl) {
                const float m = nm;
                if (j + 1 < L)
                    nm = __ldcs(a.m.proj + size_t(u0 + j + 1) * a.m.Sp + c2);
                line_sync();  // A: the updaters' partials in red
                double mine = 0;
                if (mine_lane)
#pragma unroll
                    for (int w = 0; w < NWS; ++w)
                        mine += red[w * P + lane];
                const int b = int(jl & 1);
                uint64_t* xb = &xbar[k][b];
                if (lane == 0)
                    mbar_arrive_expect_local(xb, unsigned((CL - 1) * P * sizeof(double)));
                __syncwarp();
                if (mine_lane) {
                    xred[k][b][rank][lane] = mine;
                    for (uint32_t r = 0; r < uint32_t(CL); ++r)
                        if (r != rank)
                            st_async_f64(map_peer(&xred[k][b][rank][lane], r), mine, map_peer(xb, r));
                }
                mbar_wait(xb, (jl >> 1) & 1);
                double p_bar = 0.0;  // the CTAs' partials in CTA order, the same in every CTA
                if (mine_lane)
#pragma unroll
                    for (int r = 0; r < CL; ++r)
                        p_bar += xred[k][b][r][lane];
                double factor = 0;
                if (m != 0.f && act) {
                    const double ratio = double(m) / (p_bar > pf ? p_bar : pf);
                    factor = mart_factor(ratio, a.m.beta, a.m.power);
                    if (factor <= 0) {
                        factor = pf;
                        if (rank == 0)
                            atomicAdd(a.m.clamps + c2, 1ull);
                    }
                }
                const Scale sc = GW::scale_of(factor);
                if (mine_lane)
                    fac[lane] = make_float2(sc.g, sc.lb);
                line_sync();  // B: factors in fac
                line_sync();  // C: the line's hand-overs and stores issued
                if (lane == 0)
                    st_release_cta_shared(&s_done[k], j + 1);
            }
            task = next_task(false);
        }
    } else if (lt >= GS + 64) {
        // ---- publisher warp: this CTA's part of the finished lines at gpu
        // scope (one fence + relaxed store per round; a warp of its own so the
        // fence's wait for the stores never delays the polls) ----
        const int lane = lt & 31;
        while (task < total) {
            const int sweep = task / per_sweep;
            const int v = (task % per_sweep) / nchunks, chunk = task % nchunks;
            const unsigned gs = a.epoch + unsigned(sweep);
            unsigned* mine = prog_of(v, chunk, rank);
            unsigned published = 0;
            while (published < L) {
                const unsigned d = ld_acquire_cta_shared(&s_done[k]);
                if (d > published) {
                    if (lane == 0) {
                        fence_release_gpu();
                        st_relaxed_gpu(mine, gs * L + d);
                    }
                    published = d;
                } else {
                    __nanosleep(a.pub_ns);
                }
            }
            __syncwarp();
            task = next_task(false);
        }
    } else if (lt >= GS + 32) {
        // ---- poller warp: requirements (every part of the other views'
        // progress); lane i watches line ready + i with its requirements
        // cached in registers (as the single-CTA form) ----
        constexpr int RQ = 3;
        const int lane = lt & 31;
        while (task < total) {
            const int sweep = task / per_sweep;
            const int v = (task % per_sweep) / nchunks, chunk = task % nchunks;
            const unsigned gs = a.epoch + unsigned(sweep);
            const uint32_t u0 = uint32_t(v) * L;
            if (lane < CL && gs > 0)
                spin_until_geq(prog_of(v, chunk, uint32_t(lane)), gs * L);
            __syncwarp();
            uint32_t rc[RQ], rn[RQ];
            int n = 0;
            uint32_t kx = 0, ke = 0;
            auto load_reqs = [&](unsigned j) {
                n = 0;
                kx = ke = 0;
                if (j >= L)
                    return;
                uint32_t q2 = __ldg(a.dep_off + u0 + j);
                const uint32_t e = __ldg(a.dep_off + u0 + j + 1);
                for (; q2 < e && n < RQ; ++q2) {
                    const uint32_t w = __ldg(a.deps + 2 * size_t(q2));
                    const unsigned xs = w >> 31;
                    if (gs < xs)
                        continue;
#pragma unroll
                    for (int r = 0; r < RQ; ++r)
                        if (r == n) {
                            rc[r] = uint32_t(prog_of(int(w & 0x7FFFFFFFu), chunk, 0) - a.prog);
                            rn[r] = (gs - xs) * L + __ldg(a.deps + 2 * size_t(q2) + 1);
                        }
                    ++n;
                }
                kx = q2;
                ke = e;
            };
            unsigned ready = 0, ns = 0;
            load_reqs(unsigned(lane));
            while (ready < L) {
                bool ok = true;
#pragma unroll
                for (int r = 0; r < RQ; ++r)
                    if (r < n)
#pragma unroll
                        for (int c = 0; c < CL; ++c)
                            ok = ok && ld_relaxed(a.prog + rc[r] + c * kWavePad) >= rn[r];
                for (uint32_t q2 = kx; q2 < ke && ok; ++q2) {
                    const uint32_t w = __ldg(a.deps + 2 * size_t(q2));
                    const unsigned xs = w >> 31;
                    if (gs < xs)
                        continue;
                    const unsigned need = (gs - xs) * L + __ldg(a.deps + 2 * size_t(q2) + 1);
                    const unsigned* base = prog_of(int(w & 0x7FFFFFFFu), chunk, 0);
#pragma unroll
                    for (int c = 0; c < CL; ++c)
                        ok = ok && ld_relaxed(base + c * kWavePad) >= need;
                }
                const unsigned bad = __ballot_sync(0xFFFFFFFFu, !ok);
                const unsigned adv = bad ? unsigned(__ffs(bad) - 1) : 32u;
                const unsigned nr = min(L, ready + adv);
                if (nr > ready) {
                    // acquire what the advancing lanes observed (re-reads of
                    // satisfied counters), then release to the updaters
                    fence_acquire_gpu();
                    __syncwarp();
                    ready = nr;
                    if (lane == 0)
                        st_release_cta_shared(&s_ready[k], ready);
                    const int src = lane + int(adv);
#pragma unroll
                    for (int r = 0; r < RQ; ++r) {
                        rc[r] = __shfl_sync(0xFFFFFFFFu, rc[r], src & 31);
                        rn[r] = __shfl_sync(0xFFFFFFFFu, rn[r], src & 31);
                    }
                    n = __shfl_sync(0xFFFFFFFFu, n, src & 31);
                    kx = __shfl_sync(0xFFFFFFFFu, kx, src & 31);
                    ke = __shfl_sync(0xFFFFFFFFu, ke, src & 31);
                    if (src >= 32)
                        load_reqs(ready + unsigned(lane));
                    ns = 0;
                } else {
                    ns = ns ? min(ns * 2, a.poll_ns) : 16u;
                    __nanosleep(ns);
                }
            }
            __syncwarp();
            task = next_task(false);
        }
    } else {
        // ---- updaters: the single-CTA form's line code on this CTA's cells ----
        const int t = lt;
        const int q = t % TPC, cl = t / TPC;
        float4* __restrict__ f4 = reinterpret_cast<float4*>(a.m.field);
        const uint32_t Sp4 = uint32_t(a.m.Sp) / V;
        auto wait_ready = [&](unsigned j) {
            while (ld_acquire_cta_shared(&s_ready[k]) <= j)
                __nanosleep(16);
        };
        while (task < total) {
            const int v = (task % per_sweep) / nchunks, chunk = task % nchunks;
            const uint32_t u0 = uint32_t(v) * L;
            const uint32_t col4 = (uint32_t(chunk) * P) / V + uint32_t(q);
            // a cell's float4 of this thread: fbase + cell * row_bytes (one wide
            // multiply-add per address)
            const char* const fbase = reinterpret_cast<const char*>(f4 + col4);
            const uint32_t row_bytes = Sp4 * uint32_t(sizeof(float4));
            auto cell_f4 = [&](uint32_t c) {
                return reinterpret_cast<float4*>(const_cast<char*>(fbase) + size_t(c) * row_bytes);
            };
            for (unsigned j = unsigned(t); j <= L; j += GS)
                s_pos[j] = __ldg(spos + u0 + j);
            upd_sync();
            auto load_entries = [&](unsigned j) {
                const uint32_t p0 = s_pos[j];
                const int n = int(s_pos[j + 1] - p0);
                uint2* dst = s_ent + (j % 3) * COVERL;
#pragma unroll
                for (int i = 0; i < KV; ++i) {
                    const int s = cl + i * NCLV;
                    cp_async8_if(q == 0 && s < n, dst + s, a.split + p0 + s);
                }
            };
            // a line's entries stay in registers from its copies (issued
            // during the previous line) to its scaling: one shared-memory
            // read of each per line
            uint2 enext[KV];
            auto gather = [&](unsigned j) {
                const int n = int(s_pos[j + 1] - s_pos[j]);
                const uint2* e = s_ent + (j % 3) * COVERL;
                // every entry first (the copies' asm is a compiler memory
                // barrier: reading an entry between two copies would wait for
                // each read in turn)
#pragma unroll
                for (int i = 0; i < KV; ++i) {
                    const int s = cl + i * NCLV;
                    enext[i] = s < n ? e[s] : make_uint2(kWavePrev, kWaveNoNext);
                }
#pragma unroll
                for (int i = 0; i < KV; ++i) {
                    const int s = cl + i * NCLV;
                    const uint32_t c = enext[i].x;  // bit 31: handed over, no copy
                    cp_async16_if(int(c) >= 0, buf + s * TPC + q, cell_f4(c));
                }
            };
            load_entries(0);
            if (L > 1)
                load_entries(1);
            cp_async_commit();
            cp_async_wait_all();
            upd_sync();
            wait_ready(0);
            gather(0);
            cp_async_commit();
            for (unsigned j = 0; j < L; ++j) {
                const int n = int(s_pos[j + 1] - s_pos[j]);
                uint2 ecur[KV];
#pragma unroll
                for (int i = 0; i < KV; ++i)
                    ecur[i] = enext[i];
                cp_async_wait_all();
                float4 x[KV];
#pragma unroll
                for (int i = 0; i < KV; ++i) {
                    const int s = cl + i * NCLV;
                    x[i] = s < n ? buf[s * TPC + q] : make_float4(0.f, 0.f, 0.f, 0.f);
                }
                // fp32 partials of the thread's cells and of the warp's 32 / TPC
                // threads of a problem group (at most 32 / TPC * KV cells, as
                // many as the single-CTA form's per-thread partials), fp64 from
                // the cross-warp sum on (the reference sums in fp64,
                // solver.cpp:36-40)
                float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
                for (int i = 0; i < KV; ++i) {
                    a0 += x[i].x;
                    a1 += x[i].y;
                    a2 += x[i].z;
                    a3 += x[i].w;
                }
                asm volatile("" ::"f"(a0), "f"(a1), "f"(a2), "f"(a3));
#pragma unroll
                for (int o = TPC; o < 32; o <<= 1) {
                    a0 += __shfl_xor_sync(0xFFFFFFFFu, a0, o);
                    a1 += __shfl_xor_sync(0xFFFFFFFFu, a1, o);
                    a2 += __shfl_xor_sync(0xFFFFFFFFu, a2, o);
                    a3 += __shfl_xor_sync(0xFFFFFFFFu, a3, o);
                }
                const double s0 = a0, s1 = a1, s2 = a2, s3 = a3;
                const int lane = t & 31, warp = t >> 5;
                if (lane < TPC) {
                    double* r = red + warp * P + q * V;
                    r[0] = s0;
                    r[1] = s1;
                    r[2] = s2;
                    r[3] = s3;
                }
                line_sync();  // A
                if (j + 2 < L)
                    load_entries(j + 2);
                bool issued = false;
                if (j + 1 < L && ld_acquire_cta_shared(&s_ready[k]) > j + 1) {
                    gather(j + 1);
                    issued = true;
                }
                cp_async_commit();
                line_sync();  // B
                const float4 u = reinterpret_cast<const float4*>(fac)[2 * q];
                const float4 w = reinterpret_cast<const float4*>(fac)[2 * q + 1];
                const Scale g0{u.x, u.y}, g1{u.z, u.w}, g2{w.x, w.y}, g3{w.z, w.w};
                const bool any = (u.y + u.w + w.y + w.w) != 0.f;
#pragma unroll
                for (int i = 0; i < KV; ++i) {
                    const int s = cl + i * NCLV;
                    const bool in = s < n;
                    const uint2 en = ecur[i];
                    const float4 r = GW::scale4(x[i], g0, g1, g2, g3);
                    const bool hand = in && en.y != kWaveNoNext;
                    st_shared_v4_if(hand, buf + int(en.y) * TPC + q, r);
                    st_global_cg_v4_if((any || int(en.x) < 0) && in && !hand, cell_f4(en.x & ~kWavePrev), r);
                }
                line_sync();  // C
                if (!issued && j + 1 < L) {
                    wait_ready(j + 1);
                    gather(j + 1);
                    cp_async_commit();
                }
            }
            task = next_task(false);
        }
    }
    cluster_sync_all();  // neither CTA leaves while its peer may still write its shared memory
}

template <int P, int SLOTS, int CL>
static void wave_pair_launch(const WaveArgs& a, int sms, cudaStream_t st) {
    using namespace pair;
    using SH = Shape<P, SLOTS>;
    // one CTA per SM, so that the two CTAs of a pair use two SMs' load/store
    // paths (two CTAs of one pair on one SM gain nothing): with one slot the
    // request is padded past half of the SM's shared memory
    const size_t smem = std::max<size_t>(4 * SLOTS * words<P, SLOTS>(a.lines), 120 * 1024);
    auto fn_ptr = mart_wave_pair_kernel<P, SLOTS, CL>;
    const void* fn = reinterpret_cast<const void*>(fn_ptr);
    if (smem > attr_smem(fn)) {
        UB_CUDA(cudaFuncSetAttribute(fn_ptr, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        note_attr_smem(fn, smem);
    }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(SH::NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(CL * unsigned(sms / CL));
    int clusters = 0;
    UB_CUDA(cudaOccupancyMaxActiveClusters(&clusters, fn_ptr, &cfg));
    if (clusters < 1)
        throw CudaError("mart_wave_pair_kernel cannot be resident");
    if (const char* e = std::getenv("USCG_WAVE_CLUSTERS"))
        clusters = std::max(1, std::min(clusters, std::atoi(e)));
    const int total = a.views * a.m.nchunks * a.n_sweeps;
    const int nc = std::min((total + SLOTS - 1) / SLOTS, clusters);
    cfg.gridDim = dim3(CL * unsigned(nc));
    if (const char* e = std::getenv("USCG_FLOW_VERBOSE"); e && std::atoi(e))
        std::fprintf(stderr, "mart_wave_kernel: P=%d pair cluster=%d slots=%d clusters=%d smem=%zu tasks=%d\n", P, CL,
                     SLOTS, nc, smem, total);
    // every cluster must be resident: tasks wait on smaller tickets only
    UB_CUDA(cudaLaunchKernelEx(&cfg, fn_ptr, a));
}

// CTAs per view task (USCG_WAVE_PAIR = 0 single, 1 or 2 pairs, 4 clusters of
// four forces it). Pairs pay while the pairs of the tasks in flight find SMs:
// up to four 32-problem chunks (ms per C2 iteration, pairs vs single CTA:
// 16 problems 2.42 vs 5.54, 32: 3.11 vs 4.71, 64: 3.10 vs 4.73, 128: 4.32 vs
// 4.79). Clusters of four measured slower than pairs (2.68, 3.11, 4.36 ms:
// three partial exchanges per line cost more than the halved per-CTA row
// traffic saves) and are opt-in only. Two task slots per CTA measured slower
// (6.26 ms at 128 problems, 5.53 at 32: two tasks sharing one SM's
// load/store path gain nothing) and are not dispatched.
int wave_cluster_size(const MartArgs& h) {
    const int P = h.Sp / h.nchunks;
    if (P != 16 && P != 32)
        return 1;
    if (const char* e = std::getenv("USCG_WAVE_PAIR")) {
        const int c = std::atoi(e);
        return c >= 4 ? 4 : c >= 2 ? 2 : c == 1 ? 2 : 1;
    }
    return h.Sp <= 128 ? 2 : 1;
}

bool wave_supported(const MartArgs& h) {
    int optin = 0, dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
        return false;
    const int P = h.Sp / h.nchunks;
    int cover = 0;
    switch (P) {
        case 4: cover = wave_cover<4>(); break;
        case 8: cover = wave_cover<8>(); break;
        case 16: cover = wave_cover<16>(); break;
        case 32: cover = wave_cover<32>(); break;
        default: return false;
    }
    return h.max_cells <= cover && h.max_cells < int(kWaveNoNext);
}
bool wave_fits_smem(const MartArgs& h, int lines) {
    int optin = 0, dev = 0;
    UB_CUDA(cudaGetDevice(&dev));
    UB_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    return wave_smem_bytes(h, lines) + 64 <= size_t(optin);
}

void launch_mart_wave(const MartArgs& h, const WaveSchedule& ws, unsigned* prog, unsigned* next, unsigned epoch,
                      int sweeps, cudaStream_t st, unsigned long long* prof) {
    int dev = 0, sms = 0;
    UB_CUDA(cudaGetDevice(&dev));
    UB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    if (uint64_t(ws.views) * uint64_t(h.nchunks) * uint64_t(sweeps) >= (1ull << 31) ||
        uint64_t(epoch + sweeps) * uint64_t(ws.lines) >= (1ull << 32))
        throw CudaError("mart_wave_kernel: too many tasks for one launch");
    if (!wave_supported(h) || !wave_fits_smem(h, ws.lines))
        throw CudaError("mart_wave_kernel: unsupported chunk width or line length");
    WaveArgs a;
    a.m = h;
    a.pos = ws.pos;
    a.ent = ws.ent;
    a.dep_off = ws.dep_off;
    a.deps = ws.deps;
    a.spos = ws.spos;
    a.split = ws.split;
    a.prog = prog;
    a.next = next;
    a.epoch = epoch;
    a.n_sweeps = sweeps;
    a.views = ws.views;
    a.lines = ws.lines;
    a.prof = prof;
    // field rows evict_last, traced lists evict_first (C2: 4.85 vs 4.88 ms
    // per iteration with default priorities)
    a.l2_field = 2;
    a.l2_lists = 1;
    a.poll_ns = 256;
    a.pub_ns = 32;
    if (const char* e = std::getenv("USCG_WAVE_POLL_NS"))
        a.poll_ns = unsigned(std::max(16, std::atoi(e)));
    if (const char* e = std::getenv("USCG_WAVE_PUB_NS"))
        a.pub_ns = unsigned(std::max(0, std::atoi(e)));
    if (const char* e = std::getenv("USCG_WAVE_L2")) {  // experiments: "<field><lists>" priorities
        a.l2_field = e[0] ? e[0] - '0' : 0;
        a.l2_lists = e[0] && e[1] ? e[1] - '0' : 0;
    }
    UB_CUDA(cudaMemsetAsync(next, 0, sizeof(unsigned), st));
    switch (h.Sp / h.nchunks) {
        case 4: wave_launch_t<4>(a, sms, st); break;
        case 8: wave_launch_t<8>(a, sms, st); break;
        case 16:
        case 32: {
            // (phase stamps: the single-CTA form)
            const int cl = prof || !ws.spos ? 1 : ws.parts;
            if (h.Sp / h.nchunks == 16) {
                if (cl == 2)
                    wave_pair_launch<16, 1, 2>(a, sms, st);
                else if (cl == 4)
                    wave_pair_launch<16, 1, 4>(a, sms, st);
                else
                    wave_launch_t<16>(a, sms, st);
            } else {
                if (cl == 2)
                    wave_pair_launch<32, 1, 2>(a, sms, st);
                else if (cl == 4)
                    wave_pair_launch<32, 1, 4>(a, sms, st);
                else
                    wave_launch_t<32>(a, sms, st);
            }
            break;
        }
        default: throw CudaError("mart_wave_kernel supports problem chunks of 4, 8, 16 or 32");
    }
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        throw CudaError(std::string("mart_wave_kernel launch: ") + cudaGetErrorString(e));
}

}  // namespace ub
