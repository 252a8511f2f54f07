#include "schedule.h"

#include <algorithm>

namespace ub {

void AsapSchedule::add(const uint32_t* idx, const uint32_t* pos_rel, uint32_t n) {
    level_.reserve(level_.size() + n);
    for (uint32_t u = 0; u < n; ++u) {
        const uint32_t unit = uint32_t(level_.size());
        const uint32_t b = pos_rel[u], e = pos_rel[u + 1];
        uint32_t lev = 0;
        scratch_.clear();
        for (uint32_t i = b; i < e; ++i) {
            lev = std::max(lev, last_[idx[i]]);
            const uint32_t w = writer_[idx[i]];
            if (w == kNone)
                first_cells_.push_back(idx[i]);
            else if (scratch_.empty() || scratch_.back() != w)
                scratch_.push_back(w);
        }
        first_off_.push_back(uint32_t(first_cells_.size()));
        std::sort(scratch_.begin(), scratch_.end());
        scratch_.erase(std::unique(scratch_.begin(), scratch_.end()), scratch_.end());
        preds_.insert(preds_.end(), scratch_.begin(), scratch_.end());
        pred_off_.push_back(uint32_t(preds_.size()));
        ++lev;
        for (uint32_t i = b; i < e; ++i) {
            last_[idx[i]] = lev;
            writer_[idx[i]] = unit;
        }
        level_.push_back(lev);
        max_level_ = std::max(max_level_, lev);
    }
}

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
    // cross predecessors: distinct final writers of each unit's first-touch cells
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
    // successors of p: units listing p as an in-sweep or a cross predecessor
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
    level_off.assign(size_t(max_level_) + 1, 0u);
    for (uint32_t lev : level_)
        ++level_off[lev];  // level_off[l] counts level l (1-based) for now
    // exclusive offsets: level l (1-based) occupies [level_off[l-1], level_off[l])
    uint32_t acc = 0;
    std::vector<uint32_t> start(size_t(max_level_) + 1, 0u);
    for (uint32_t l = 1; l <= max_level_; ++l) {
        start[l] = acc;
        acc += level_off[l];
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
