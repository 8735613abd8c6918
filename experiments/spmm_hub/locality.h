// Locality schedule of the wide local SpMM (host side, built once per part at cdfgnn_init).
//
// PAPER.md §4 renumbers each subgraph's vertices "for continuous memory
// access"; on B200 the gather SpMM Z̈ = Â_i T is bound by L2->SM delivery of neighbour rows
// (every non-zero re-reads a row of T), so the renumbering here is chosen for reuse:
//   1. label propagation (asynchronous, ascending row order, ties kept / to the smaller label,
//      deterministic) groups the rows into communities — label-free, from the graph alone;
//   2. rows are ordered by (community, degree descending, row id); the first H members of
//      each community are its hub rows;
//   3. every row's neighbour list is rewritten in the new ids with the neighbours inside its
//      community's hub range first.
// The kernel (kernels_spmm.cu, spmm_hub) stages one column slice of a community's hub rows
// in shared memory and serves those neighbours from it; the ABI's local row order (R21), the
// CSR the caller sees and the oracle are unchanged — only the SpMM's internal copy of T is
// stored in the new order.
#pragma once
#include <cstdint>
#include <vector>

namespace cdfgnn {

struct HubSchedule {
    int64_t n = 0, nnz = 0;
    int32_t hub_rows = 0;                 // H: hub rows staged per (community, slice)
    std::vector<int32_t> order;           // [n] new id -> local row
    std::vector<int32_t> rowptr;          // [n+1] CSR in new row order
    std::vector<int32_t> nhub;            // [n] neighbours of the row inside its hub range (listed first)
    std::vector<int32_t> col;             // [nnz] neighbour new ids
    std::vector<float> val;               // [nnz] Â weights, same order
    // one entry per community, heaviest first: {first row, end row, hub base (new id), hub count}
    std::vector<int32_t> comm;            // [4 * communities]
    int32_t communities = 0;
    double in_comm_frac = 0.0;            // share of non-zeros inside their row's community
    double hub_frac = 0.0;                // share of non-zeros served from the hub rows
    int lpa_iters = 0;
};

// rowptr/colidx/val: the part's local CSR (n rows).  hub_rows: H.
void build_hub_schedule(int64_t n, const int32_t* rowptr, const int32_t* colidx, const float* val,
                        int32_t hub_rows, HubSchedule& out);

}  // namespace cdfgnn
