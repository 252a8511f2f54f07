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
    explicit AsapSchedule(uint64_t cell_count)
        : last_(cell_count, 0u), writer_(cell_count, kNone) {}

    // supports of consecutive units in sweep order, CSR over `pos`
    // (pos[i]..pos[i+1] relative to idx), units u0 .. u0+n-1
    void add(const uint32_t* idx, const uint32_t* pos_rel, uint32_t n);

    // counting sort of the units by level: order (units), level_off (levels + 1)
    void finish(std::vector<uint32_t>& order, std::vector<uint32_t>& level_off) const;

    // Direct predecessors of every unit (by unit id): the distinct units that
    // last wrote one of its cells earlier in the sweep. A unit may run as
    // soon as all of them are done (dataflow execution of the same order).
    const std::vector<uint32_t>& pred_off() const { return pred_off_; }
    const std::vector<uint32_t>& preds() const { return preds_; }

    // successors (transpose of preds): succ_off (units + 1), succs
    void successors(std::vector<uint32_t>& succ_off, std::vector<uint32_t>& succs) const;

    // Cross-sweep dependencies (for sweeps run back to back): a unit's
    // cross predecessors are the final writers, in the previous sweep, of the
    // cells it is the first in its sweep to touch. npred_x (units) counts
    // them; succ_all merges in- and cross-successors (a unit can appear in
    // both lists, it is then counted once for each).
    void cross(std::vector<uint32_t>& npred_x, std::vector<uint32_t>& succ_all_off,
               std::vector<uint32_t>& succ_all) const;

    uint32_t levels() const { return max_level_; }

    static constexpr uint32_t kNone = 0xFFFFFFFFu;

private:
    std::vector<uint32_t> last_;    // level of the last writer per cell
    std::vector<uint32_t> writer_;  // unit id of the last writer per cell
    std::vector<uint32_t> level_;
    std::vector<uint32_t> pred_off_{0u};
    std::vector<uint32_t> preds_;
    std::vector<uint32_t> first_off_{0u};  // per unit: cells it touches first in the sweep
    std::vector<uint32_t> first_cells_;
    std::vector<uint32_t> scratch_;
    uint32_t max_level_ = 0;
};

}  // namespace ub
