#include "schedule.h"

#include <algorithm>

namespace ub {

AsapSchedule::AsapSchedule(uint64_t cell_count, uint32_t lines_per_view, uint32_t run)
    : lines_per_view_(lines_per_view ? lines_per_view : 1), run_(run ? run : 1),
      writer_(cell_count, kNone) {
    runs_per_view_ = (lines_per_view_ + run_ - 1) / run_;
}

void AsapSchedule::close_run() {
    if (cur_run_ == kNone)
        return;
    std::sort(scratch_.begin(), scratch_.end());
    scratch_.erase(std::unique(scratch_.begin(), scratch_.end()), scratch_.end());
    uint32_t lev = 0;
    for (uint32_t p : scratch_)
        lev = std::max(lev, level_[p]);
    ++lev;
    preds_.insert(preds_.end(), scratch_.begin(), scratch_.end());
    pred_off_.push_back(uint32_t(preds_.size()));
    first_off_.push_back(uint32_t(first_cells_.size()));
    level_.push_back(lev);
    max_level_ = std::max(max_level_, lev);
    scratch_.clear();
    cur_run_ = kNone;
}

void AsapSchedule::add(const uint32_t* idx, const uint32_t* pos_rel, uint32_t n) {
    for (uint32_t i = 0; i < n; ++i, ++lines_added_) {
        const uint64_t u = lines_added_;
        const uint32_t run = uint32_t((u / lines_per_view_) * runs_per_view_ +
                                      (u % lines_per_view_) / run_);
        if (run != cur_run_) {
            close_run();
            cur_run_ = run;  // runs arrive in id order: run == level_.size()
        }
        for (uint32_t k = pos_rel[i]; k < pos_rel[i + 1]; ++k) {
            const uint32_t c = idx[k];
            const uint32_t w = writer_[c];
            if (w == run)
                continue;  // written by an earlier line of this run
            if (w == kNone)
                first_cells_.push_back(c);
            else if (scratch_.empty() || scratch_.back() != w)
                scratch_.push_back(w);
            writer_[c] = run;
        }
    }
}

void AsapSchedule::done() { close_run(); }

void AsapSchedule::successors(std::vector<uint32_t>& succ_off,
                              std::vector<uint32_t>& succs) const {
    const size_t units = level_.size();
    succ_off.assign(units + 1, 0u);
    for (uint32_t p : preds_)
        ++succ_off[p + 1];
    for (size_t u = 0; u < units; ++u)
        succ_off[u + 1] += succ_off[u];
    succs.assign(preds_.size(), 0u);
    std::vector<uint32_t> cur(succ_off.begin(), succ_off.end() - 1);
    for (size_t u = 0; u < units; ++u)
        for (uint32_t k = pred_off_[u]; k < pred_off_[u + 1]; ++k)
            succs[cur[preds_[k]]++] = uint32_t(u);
}

void AsapSchedule::cross(std::vector<uint32_t>& npred_x, std::vector<uint32_t>& succ_all_off,
                         std::vector<uint32_t>& succ_all) const {
    const size_t units = level_.size();
    // cross predecessors: distinct final writers of each run's first-touch cells
    std::vector<uint32_t> xoff(units + 1, 0u), xpred;
    std::vector<uint32_t> tmp;
    for (size_t u = 0; u < units; ++u) {
        tmp.clear();
        for (uint32_t k = first_off_[u]; k < first_off_[u + 1]; ++k)
            tmp.push_back(writer_[first_cells_[k]]);
        std::sort(tmp.begin(), tmp.end());
        tmp.erase(std::unique(tmp.begin(), tmp.end()), tmp.end());
        xpred.insert(xpred.end(), tmp.begin(), tmp.end());
        xoff[u + 1] = uint32_t(xpred.size());
    }
    npred_x.assign(units, 0u);
    for (size_t u = 0; u < units; ++u)
        npred_x[u] = xoff[u + 1] - xoff[u];
    // successors of p: runs listing p as an in-sweep or a cross-sweep predecessor
    succ_all_off.assign(units + 1, 0u);
    for (uint32_t p : preds_)
        ++succ_all_off[p + 1];
    for (uint32_t p : xpred)
        ++succ_all_off[p + 1];
    for (size_t u = 0; u < units; ++u)
        succ_all_off[u + 1] += succ_all_off[u];
    succ_all.assign(preds_.size() + xpred.size(), 0u);
    std::vector<uint32_t> cur(succ_all_off.begin(), succ_all_off.end() - 1);
    for (size_t u = 0; u < units; ++u) {
        for (uint32_t k = pred_off_[u]; k < pred_off_[u + 1]; ++k)
            succ_all[cur[preds_[k]]++] = uint32_t(u);
        for (uint32_t k = xoff[u]; k < xoff[u + 1]; ++k)
            succ_all[cur[xpred[k]]++] = uint32_t(u);
    }
}

void AsapSchedule::finish(std::vector<uint32_t>& order, std::vector<uint32_t>& level_off) const {
    std::vector<uint32_t> cnt(size_t(max_level_) + 1, 0u);
    for (uint32_t lev : level_)
        ++cnt[lev];
    // level l (1-based) occupies [start[l], start[l] + cnt[l])
    std::vector<uint32_t> start(size_t(max_level_) + 1, 0u);
    uint32_t acc = 0;
    for (uint32_t l = 1; l <= max_level_; ++l) {
        start[l] = acc;
        acc += cnt[l];
    }
    order.assign(level_.size(), 0u);
    std::vector<uint32_t> cur(start);
    for (uint32_t u = 0; u < level_.size(); ++u)
        order[cur[level_[u]]++] = u;  // stable: sweep order inside a level
    level_off.assign(size_t(max_level_) + 1, 0u);
    for (uint32_t l = 1; l <= max_level_; ++l)
        level_off[l - 1] = start[l];
    level_off[max_level_] = acc;
}

}  // namespace ub
