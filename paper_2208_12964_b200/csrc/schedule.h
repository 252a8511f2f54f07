// MART dependency schedule (host C++).
//
// The reference's Sp-MART is a strictly sequential row action
// (proj/src/solver.cpp:111-136, proj/README.md:84-86): line (v, l) reads the
// field as left by every earlier line. Two lines commute when their cell
// supports are disjoint, so the ASAP level of a line in sweep order,
//     level(u) = 1 + max_{c in support(u)} last[c],   then last[c] = level(u),
// groups lines into levels whose members are pairwise disjoint and whose
// per-cell order matches the sweep order. Executing level after level
// therefore reproduces the sequential result exactly (up to the fp32 field).
// The schedule depends on geometry only, so it is built once per tracer.
#pragma once

#include <cstdint>
#include <vector>

namespace ub {

class AsapSchedule {
public:
    explicit AsapSchedule(uint64_t cell_count) : last_(cell_count, 0u) {}

    // supports of consecutive units in sweep order, CSR over `pos`
    // (pos[i]..pos[i+1] relative to idx), units u0 .. u0+n-1
    void add(const uint32_t* idx, const uint32_t* pos_rel, uint32_t n);

    // counting sort of the units by level: order (units), level_off (levels + 1)
    void finish(std::vector<uint32_t>& order, std::vector<uint32_t>& level_off) const;

    uint32_t levels() const { return max_level_; }

private:
    std::vector<uint32_t> last_;
    std::vector<uint32_t> level_;
    uint32_t max_level_ = 0;
};

}  // namespace ub
