// Locality schedule of the wide local SpMM (see locality.h).
#include "locality.h"

#include <algorithm>
#include <climits>
#include <numeric>

namespace cdfgnn {

namespace {

// Asynchronous label propagation in ascending row order: every row takes the label most
// frequent among its neighbours, keeping its own label when that ties the maximum, else the
// smallest of the tied labels.  Stops when fewer than n/1000 rows change (<= 12 passes).
int label_propagation(int64_t n, const int32_t* rowptr, const int32_t* colidx, std::vector<int32_t>& lab) {
    lab.resize(n);
    std::iota(lab.begin(), lab.end(), 0);
    std::vector<int32_t> cnt(n, 0), touched;
    int it = 0;
    for (; it < 12; ++it) {
        int64_t changed = 0;
        for (int64_t v = 0; v < n; ++v) {
            touched.clear();
            for (int64_t e = rowptr[v]; e < rowptr[v + 1]; ++e) {
                const int32_t l = lab[colidx[e]];
                if (cnt[l]++ == 0) touched.push_back(l);
            }
            int32_t bc = 0;
            for (int32_t l : touched) bc = std::max(bc, cnt[l]);
            int32_t best = lab[v];
            if (cnt[lab[v]] < bc) {
                best = INT32_MAX;
                for (int32_t l : touched)
                    if (cnt[l] == bc && l < best) best = l;
            }
            for (int32_t l : touched) cnt[l] = 0;
            if (best != lab[v]) {
                lab[v] = best;
                ++changed;
            }
        }
        if (changed * 1000 < n) {
            ++it;
            break;
        }
    }
    return it;
}

}  // namespace

void build_hub_schedule(int64_t n, const int32_t* rowptr, const int32_t* colidx, const float* val,
                        int32_t hub_rows, HubSchedule& out) {
    out = HubSchedule{};
    out.n = n;
    out.nnz = n ? rowptr[n] : 0;
    out.hub_rows = hub_rows;
    if (n == 0) return;
    std::vector<int32_t> lab;
    out.lpa_iters = label_propagation(n, rowptr, colidx, lab);
    // compact community ids, ordered by first appearance
    std::vector<int32_t> cid(n, -1);
    int32_t nc = 0;
    for (int64_t v = 0; v < n; ++v) {
        if (cid[lab[v]] < 0) cid[lab[v]] = nc++;
    }
    std::vector<int32_t> com(n);
    for (int64_t v = 0; v < n; ++v) com[v] = cid[lab[v]];
    // rows by (community, degree desc, row id)
    out.order.resize(n);
    std::iota(out.order.begin(), out.order.end(), 0);
    std::stable_sort(out.order.begin(), out.order.end(), [&](int32_t a, int32_t b) {
        if (com[a] != com[b]) return com[a] < com[b];
        return rowptr[a + 1] - rowptr[a] > rowptr[b + 1] - rowptr[b];
    });
    std::vector<int32_t> inv(n);
    for (int64_t i = 0; i < n; ++i) inv[out.order[i]] = (int32_t)i;
    // community ranges and hub ranges (new ids)
    std::vector<int32_t> cb(nc + 1, 0);
    for (int64_t i = 0; i < n; ++i) cb[com[out.order[i]] + 1]++;
    for (int32_t c = 0; c < nc; ++c) cb[c + 1] += cb[c];
    // CSR in new row order, hub neighbours first
    out.rowptr.assign(n + 1, 0);
    out.nhub.assign(n, 0);
    out.col.resize(out.nnz);
    out.val.resize(out.nnz);
    int64_t inside = 0, hubs = 0, pos = 0;
    std::vector<int64_t> work(nc, 0);
    for (int64_t i = 0; i < n; ++i) {
        const int32_t r = out.order[i];
        const int32_t c = com[r];
        const int32_t hb = cb[c], he = cb[c] + std::min<int32_t>(hub_rows, cb[c + 1] - cb[c]);
        out.rowptr[i] = (int32_t)pos;
        int64_t k = pos;
        for (int64_t e = rowptr[r]; e < rowptr[r + 1]; ++e) {
            const int32_t j = inv[colidx[e]];
            if (j >= hb && j < he) {
                out.col[k] = j;
                out.val[k] = val[e];
                ++k;
            }
        }
        out.nhub[i] = (int32_t)(k - pos);
        for (int64_t e = rowptr[r]; e < rowptr[r + 1]; ++e) {
            const int32_t j = inv[colidx[e]];
            if (!(j >= hb && j < he)) {
                out.col[k] = j;
                out.val[k] = val[e];
                ++k;
            }
            inside += com[colidx[e]] == c;
        }
        hubs += out.nhub[i];
        work[c] += rowptr[r + 1] - rowptr[r] + 1;
        pos = k;
    }
    out.rowptr[n] = (int32_t)pos;
    // communities heaviest first (the kernel takes (community, slice) units in this order)
    std::vector<int32_t> cs(nc);
    std::iota(cs.begin(), cs.end(), 0);
    std::stable_sort(cs.begin(), cs.end(), [&](int32_t a, int32_t b) { return work[a] > work[b]; });
    out.communities = nc;
    out.comm.resize(4 * (size_t)nc);
    for (int32_t t = 0; t < nc; ++t) {
        const int32_t c = cs[t];
        out.comm[4 * t + 0] = cb[c];
        out.comm[4 * t + 1] = cb[c + 1];
        out.comm[4 * t + 2] = cb[c];
        out.comm[4 * t + 3] = std::min<int32_t>(hub_rows, cb[c + 1] - cb[c]);
    }
    out.in_comm_frac = out.nnz ? (double)inside / (double)out.nnz : 0.0;
    out.hub_frac = out.nnz ? (double)hubs / (double)out.nnz : 0.0;
}

}  // namespace cdfgnn
