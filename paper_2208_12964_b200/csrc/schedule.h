// MART dependency schedule (host C++).
//
// The reference's Sp-MART is a strictly sequential row action
// (proj/src/solver.cpp:111-136, proj/README.md:84-86): line (v, l) reads the
// field as left by every earlier line. Two lines commute when their cell
// supports are disjoint. Lines are grouped into runs ("macro units") of R
// consecutive lines of one view; a run is contiguous in sweep order, so the
// runs form a DAG (no cycles) whose edges are exactly the line dependencies
// that cross runs. For every run:
//   preds  = distinct runs that last wrote one of its cells before it,
//   level  = 1 + max level of its preds (ASAP),
// and, for sweeps run back to back, its cross-sweep preds = the final writers
// (previous sweep) of the cells it is the first in its sweep to touch.
// Running every run after its preds, its lines in order, performs on every
// cell exactly the reference's sequence of updates. R = 1 is the line DAG.
// The schedule depends on geometry only, so it is built once per tracer.
#pragma once

#include <cstdint>
#include <vector>

namespace ub {

class AsapSchedule {
public:
    // lines_per_view: runs never cross a view; run: lines per run (>= 1)
    AsapSchedule(uint64_t cell_count, uint32_t lines_per_view, uint32_t run);

    // supports of consecutive lines in sweep order, CSR over pos_rel
    // (pos_rel[i]..pos_rel[i+1] relative to idx), n lines
    void add(const uint32_t* idx, const uint32_t* pos_rel, uint32_t n);
    // finalize the last run (call after the last add)
    void done();

    // counting sort of the runs by level: order (runs), level_off (levels + 1)
    void finish(std::vector<uint32_t>& order, std::vector<uint32_t>& level_off) const;

    const std::vector<uint32_t>& pred_off() const { return pred_off_; }
    const std::vector<uint32_t>& preds() const { return preds_; }

    // successors (transpose of preds): succ_off (runs + 1), succs
    void successors(std::vector<uint32_t>& succ_off, std::vector<uint32_t>& succs) const;

    // cross-sweep predecessor counts and merged in-/cross-sweep successors
    void cross(std::vector<uint32_t>& npred_x, std::vector<uint32_t>& succ_all_off,
               std::vector<uint32_t>& succ_all) const;

    uint32_t levels() const { return max_level_; }
    uint32_t runs() const { return uint32_t(level_.size()); }
    uint32_t runs_per_view() const { return runs_per_view_; }

    static constexpr uint32_t kNone = 0xFFFFFFFFu;

private:
    void close_run();

    uint32_t lines_per_view_, run_, runs_per_view_;
    uint64_t lines_added_ = 0;
    std::vector<uint32_t> writer_;  // run id of the last writer per cell
    std::vector<uint32_t> level_;   // per run
    std::vector<uint32_t> pred_off_{0u};
    std::vector<uint32_t> preds_;
    std::vector<uint32_t> first_off_{0u};  // per run: cells it touches first in the sweep
    std::vector<uint32_t> first_cells_;
    std::vector<uint32_t> scratch_;
    std::vector<uint32_t> pending_cells_;  // cells of the open run (written at close)
    uint32_t cur_run_ = kNone;
    uint32_t max_level_ = 0;
};

}  // namespace ub
