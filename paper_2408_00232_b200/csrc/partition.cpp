// Hierarchical EBV vertex-cut partitioner and partition plan (host C++).
//
// PAPER.md §6: edges are assigned one by one to the part that
// minimises
//   Eva_(u,v)(i) = (1-γ)(𝟙[i∉d_rep_u] + 𝟙[i∉d_rep_v]) + γ(𝟙[host_i∉h_rep_u] + 𝟙[host_i∉h_rep_v])
//                + α e_count[i]/(|E|/p) + β v_count[i]/(|V|/p)
// Scores are compared exactly: multiplied by gd·ad·bd·|E|·|V| they are integers
// (γ = gn/gd, α = an/ad, β = bn/bd), kept incrementally per part in __int128.
// Ties go to the lowest part id; a vertex's master is the first part it is
// assigned to; isolated vertices go to argmin v_count after all edges (R20).
// Local order (R21): [boundary masters ↑gid][mirrors by master part ↑, ↑gid][interior ↑gid].
// Â_i weights 1/sqrt(d_u d_v) use GLOBAL degrees (R2), computed in double
// and rounded once to fp32.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <thread>
#include <vector>

#include "common.h"

namespace {

using i128 = __int128;

struct PartData {
    int32_t part = 0;
    int64_t n_local = 0, B = 0, M = 0, n_edges = 0;
    std::vector<int32_t> l2g, rowptr, colidx, halo_local;
    std::vector<float> val;
    std::vector<int64_t> moff, hoff;
};

inline uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// LSD radix sort of (key, payload) by 64-bit key; stable.
void radix_sort_u64(std::vector<uint64_t>& key, std::vector<int64_t>& idx) {
    const size_t n = key.size();
    std::vector<uint64_t> k2(n);
    std::vector<int64_t> i2(n);
    for (int shift = 0; shift < 64; shift += 16) {
        // skip passes whose digit is constant
        uint64_t first = n ? (key[0] >> shift) & 0xFFFF : 0;
        bool constant = true;
        for (size_t t = 0; t < n && constant; ++t)
            if (((key[t] >> shift) & 0xFFFF) != first) constant = false;
        if (constant) continue;
        std::vector<size_t> cnt(65537, 0);
        for (size_t t = 0; t < n; ++t) cnt[((key[t] >> shift) & 0xFFFF) + 1]++;
        for (int b = 0; b < 65536; ++b) cnt[b + 1] += cnt[b];
        for (size_t t = 0; t < n; ++t) {
            size_t d = cnt[(key[t] >> shift) & 0xFFFF]++;
            k2[d] = key[t];
            i2[d] = idx[t];
        }
        key.swap(k2);
        idx.swap(i2);
    }
}

}  // namespace

struct cdfgnn_plan {
    int64_t n = 0, m = 0;
    int32_t p = 0;
    std::vector<int32_t> host;
    std::vector<PartData> parts;
    cdfgnn_partition_stats stats{};
};

extern "C" int cdfgnn_partition_cfg_default(cdfgnn_partition_cfg* cfg, int32_t p) {
    if (!cfg) CDF_FAIL(CDFGNN_EUSAGE, "cfg is NULL");
    std::memset(cfg, 0, sizeof(*cfg));
    cfg->num_parts = p;
    cfg->num_hosts = 1;
    cfg->host_of = nullptr;
    cfg->alpha_num = 1; cfg->alpha_den = 1;
    cfg->beta_num = 1; cfg->beta_den = 1;
    cfg->gamma_num = 1; cfg->gamma_den = 10;
    cfg->edge_order = 1;
    cfg->seed = 0;
    cfg->self_loops = 0;
    return CDFGNN_OK;
}

extern "C" int cdfgnn_partition(int64_t n, int64_t m, const int32_t* eu, const int32_t* ev,
                                const cdfgnn_partition_cfg* cfg, int32_t* edge_part_out,
                                int32_t* master_out, cdfgnn_plan** plan_out) {
    if (!cfg || !plan_out) CDF_FAIL(CDFGNN_EUSAGE, "cfg and plan must be non-NULL");
    *plan_out = nullptr;
    const int32_t p = cfg->num_parts;
    if (p < 1 || p > CDFGNN_MAX_PARTS) CDF_FAIL(CDFGNN_EUSAGE, "num_parts must be in [1, 64], got %d", p);
    if (m <= 0) CDF_FAIL(CDFGNN_EUSAGE, "the graph has no edges");
    if (n <= 0 || n > INT32_MAX) CDF_FAIL(CDFGNN_EUSAGE, "n must be in [1, 2^31)");
    if (!eu || !ev) CDF_FAIL(CDFGNN_EUSAGE, "edge arrays are NULL");
    if (cfg->alpha_den <= 0 || cfg->beta_den <= 0 || cfg->gamma_den <= 0 || cfg->gamma_num < 0 ||
        cfg->gamma_num > cfg->gamma_den || cfg->alpha_num < 0 || cfg->beta_num < 0)
        CDF_FAIL(CDFGNN_EUSAGE, "alpha/beta/gamma must be non-negative fractions with gamma <= 1");
    const int32_t nh = cfg->num_hosts < 1 ? 1 : cfg->num_hosts;
    if (nh > 64) CDF_FAIL(CDFGNN_EUSAGE, "num_hosts must be <= 64");
    std::vector<int32_t> host(p);
    for (int i = 0; i < p; ++i) {
        host[i] = cfg->host_of ? cfg->host_of[i] : (int32_t)((int64_t)i * nh / p);
        if (host[i] < 0 || host[i] >= 64) CDF_FAIL(CDFGNN_EUSAGE, "host id out of range");
    }
    // ---- validate: ids in range, no self-loop, no duplicate (S:L50 semantics)
    std::vector<uint64_t> key(m);
    std::vector<int64_t> idx(m);
    for (int64_t e = 0; e < m; ++e) {
        int64_t u = eu[e], v = ev[e];
        if (u < 0 || v < 0 || u >= n || v >= n)
            CDF_FAIL(CDFGNN_EDATA, "edge %lld endpoint out of range", (long long)e);
        if (u == v) CDF_FAIL(CDFGNN_EDATA, "edge %lld is a self-loop", (long long)e);
        uint64_t a = (uint64_t)std::min(u, v), b = (uint64_t)std::max(u, v);
        key[e] = (a << 32) | b;
        idx[e] = e;
    }
    radix_sort_u64(key, idx);
    for (int64_t t = 1; t < m; ++t)
        if (key[t] == key[t - 1]) CDF_FAIL(CDFGNN_EDATA, "duplicate edge %lld", (long long)idx[t]);
    std::vector<int64_t> deg(n, 0);
    for (int64_t e = 0; e < m; ++e) { deg[eu[e]]++; deg[ev[e]]++; }
    // ---- streaming order (reading R19)
    std::vector<int64_t> order;
    if (cfg->edge_order == 0) {
        order.resize(m);
        std::iota(order.begin(), order.end(), 0);
    } else if (cfg->edge_order == 1) {
        // idx is sorted by (min, max); stable counting sort by d_u + d_v
        int64_t maxs = 0;
        for (int64_t e = 0; e < m; ++e) maxs = std::max(maxs, deg[eu[e]] + deg[ev[e]]);
        std::vector<int64_t> cnt(maxs + 2, 0);
        for (int64_t t = 0; t < m; ++t) cnt[deg[eu[idx[t]]] + deg[ev[idx[t]]] + 1]++;
        for (int64_t s = 0; s <= maxs; ++s) cnt[s + 1] += cnt[s];
        order.resize(m);
        for (int64_t t = 0; t < m; ++t) {
            int64_t e = idx[t];
            order[cnt[deg[eu[e]] + deg[ev[e]]]++] = e;
        }
    } else if (cfg->edge_order == 2) {
        std::vector<uint64_t> k(m);
        std::vector<int64_t> o(m);
        for (int64_t e = 0; e < m; ++e) {
            k[e] = splitmix64(cfg->seed ^ ((uint64_t)e * 0xD1B54A32D192ED03ull));
            o[e] = e;
        }
        radix_sort_u64(k, o);
        order.swap(o);
    } else {
        CDF_FAIL(CDFGNN_EUSAGE, "edge_order must be 0, 1 or 2");
    }
    key.clear(); key.shrink_to_fit();
    idx.clear(); idx.shrink_to_fit();
    // ---- the greedy streaming loop
    const i128 E = m, V = n;
    const i128 gn = cfg->gamma_num, gd = cfg->gamma_den, an = cfg->alpha_num,
               ad = cfg->alpha_den, bn = cfg->beta_num, bd = cfg->beta_den;
    const i128 c_rep = (gd - gn) * ad * bd * E * V;
    const i128 c_host = gn * ad * bd * E * V;
    const i128 c_e = an * gd * bd * (i128)p * V;
    const i128 c_v = bn * gd * ad * (i128)p * E;
    std::vector<uint64_t> d_rep(n, 0), h_rep(n, 0);
    std::vector<int64_t> e_count(p, 0), v_count(p, 0);
    std::vector<i128> bal(p, 0);   // c_e e_count[i] + c_v v_count[i]
    std::vector<int32_t> master(n, -1);
    std::vector<int32_t> epart(m);
    std::vector<uint64_t> hbit(p);
    for (int i = 0; i < p; ++i) hbit[i] = 1ull << host[i];
    for (int64_t t = 0; t < m; ++t) {
        const int64_t e = order[t];
        const int32_t u = eu[e], v = ev[e];
        const uint64_t du = d_rep[u], dv = d_rep[v], hu = h_rep[u], hv = h_rep[v];
        i128 best = 0;
        int bi = 0;
        for (int i = 0; i < p; ++i) {
            const uint64_t b = 1ull << i;
            const int rep = !(du & b) + !(dv & b);
            const int hst = !(hu & hbit[i]) + !(hv & hbit[i]);
            const i128 s = c_rep * rep + c_host * hst + bal[i];
            if (i == 0 || s < best) { best = s; bi = i; }
        }
        epart[e] = bi;
        e_count[bi]++;
        bal[bi] += c_e;
        const uint64_t b = 1ull << bi;
        for (int32_t x : {u, v}) {
            if (!(d_rep[x] & b)) {
                d_rep[x] |= b;
                v_count[bi]++;
                bal[bi] += c_v;
                if (master[x] < 0) master[x] = bi;
            }
            h_rep[x] |= hbit[bi];
        }
    }
    for (int64_t x = 0; x < n; ++x) {
        if (master[x] < 0) {
            int bi = 0;
            for (int i = 1; i < p; ++i)
                if (v_count[i] < v_count[bi]) bi = i;
            master[x] = bi;
            d_rep[x] |= 1ull << bi;
            v_count[bi]++;
        }
    }
    order.clear(); order.shrink_to_fit();
    // ---- plan (reading R21)
    auto* plan = new cdfgnn_plan();
    plan->n = n; plan->m = m; plan->p = p; plan->host = host;
    plan->parts.resize(p);
    // mirrors[i][j]: vertices mastered on j with a mirror on i, ascending gid
    std::vector<std::vector<std::vector<int32_t>>> mir(p, std::vector<std::vector<int32_t>>(p));
    std::vector<std::vector<int32_t>> bm(p), inter(p);
    for (int64_t x = 0; x < n; ++x) {
        const uint64_t r = d_rep[x];
        const int mx = master[x];
        const bool boundary = (r & (r - 1)) != 0;
        for (uint64_t rr = r; rr; rr &= rr - 1) {
            const int i = __builtin_ctzll(rr);
            if (i == mx) (boundary ? bm[i] : inter[i]).push_back((int32_t)x);
            else mir[i][mx].push_back((int32_t)x);
        }
    }
    std::vector<std::vector<int32_t>> g2l(p);
    for (int i = 0; i < p; ++i) {
        PartData& P = plan->parts[i];
        P.part = i;
        P.B = (int64_t)bm[i].size();
        P.moff.assign(p + 1, 0);
        P.l2g = bm[i];
        for (int j = 0; j < p; ++j) {
            P.moff[j + 1] = P.moff[j] + (int64_t)mir[i][j].size();
            P.l2g.insert(P.l2g.end(), mir[i][j].begin(), mir[i][j].end());
        }
        P.M = P.moff[p];
        P.l2g.insert(P.l2g.end(), inter[i].begin(), inter[i].end());
        P.n_local = (int64_t)P.l2g.size();
        g2l[i].assign(n, -1);
        for (int64_t k = 0; k < P.n_local; ++k) g2l[i][P.l2g[k]] = (int32_t)k;
    }
    for (int j = 0; j < p; ++j) {
        PartData& P = plan->parts[j];
        P.hoff.assign(p + 1, 0);
        for (int s = 0; s < p; ++s) {
            P.hoff[s + 1] = P.hoff[s] + (s == j ? 0 : (int64_t)mir[s][j].size());
            if (s != j)
                for (int32_t x : mir[s][j]) P.halo_local.push_back(g2l[j][x]);
        }
    }
    // ---- per-part CSR of Â_i (both directions of every assigned edge; + loops)
    std::vector<std::vector<int64_t>> part_edges(p);
    for (int64_t e = 0; e < m; ++e) part_edges[epart[e]].push_back(e);
    auto build_csr = [&](int i) {
        PartData& P = plan->parts[i];
        const std::vector<int32_t>& gl = g2l[i];
        const auto& pe = part_edges[i];
        P.n_edges = (int64_t)pe.size();
        const int64_t nl = P.n_local;
        int64_t loops = cfg->self_loops ? (P.B + (int64_t)inter[i].size()) : 0;
        const int64_t nnz = 2 * P.n_edges + loops;
        if (nnz >= INT32_MAX) return;  // checked below
        std::vector<int32_t> r(nnz), c(nnz);
        int64_t k = 0;
        for (int64_t e : pe) {
            int32_t a = gl[eu[e]], b = gl[ev[e]];
            r[k] = a; c[k] = b; ++k;
            r[k] = b; c[k] = a; ++k;
        }
        if (cfg->self_loops) {
            for (int64_t x = 0; x < P.B; ++x) { r[k] = (int32_t)x; c[k] = (int32_t)x; ++k; }
            for (int64_t x = P.B + P.M; x < nl; ++x) { r[k] = (int32_t)x; c[k] = (int32_t)x; ++k; }
        }
        // counting sort by column, then stable by row -> (row, col) ascending
        std::vector<int64_t> cnt(nl + 1, 0);
        for (int64_t t = 0; t < nnz; ++t) cnt[c[t] + 1]++;
        for (int64_t x = 0; x < nl; ++x) cnt[x + 1] += cnt[x];
        std::vector<int32_t> r2(nnz), c2(nnz);
        for (int64_t t = 0; t < nnz; ++t) {
            int64_t d = cnt[c[t]]++;
            r2[d] = r[t]; c2[d] = c[t];
        }
        std::vector<int32_t>().swap(r);
        std::vector<int32_t>().swap(c);
        P.rowptr.assign(nl + 1, 0);
        for (int64_t t = 0; t < nnz; ++t) P.rowptr[r2[t] + 1]++;
        for (int64_t x = 0; x < nl; ++x) P.rowptr[x + 1] += P.rowptr[x];
        std::vector<int64_t> fill(P.rowptr.begin(), P.rowptr.end() - 1);
        P.colidx.resize(nnz);
        P.val.resize(nnz);
        for (int64_t t = 0; t < nnz; ++t) {
            int64_t d = fill[r2[t]]++;
            P.colidx[d] = c2[t];
            const int64_t gu = P.l2g[r2[t]], gv = P.l2g[c2[t]];
            const double du = (double)(deg[gu] + (cfg->self_loops ? 1 : 0));
            const double dv = (double)(deg[gv] + (cfg->self_loops ? 1 : 0));
            P.val[d] = (float)(1.0 / std::sqrt(du * dv));
        }
    };
    for (int i = 0; i < p; ++i)
        if (2 * (int64_t)part_edges[i].size() + n >= INT32_MAX) {
            delete plan;
            CDF_FAIL(CDFGNN_EUSAGE, "part %d has too many CSR entries for int32 indices", i);
        }
    {
        std::vector<std::thread> th;
        const int nt = std::max(1, std::min<int>(p, (int)std::thread::hardware_concurrency()));
        for (int w = 0; w < nt; ++w)
            th.emplace_back([&, w]() {
                for (int i = w; i < p; i += nt) build_csr(i);
            });
        for (auto& t : th) t.join();
    }
    // ---- statistics
    cdfgnn_partition_stats& st = plan->stats;
    int64_t sum_vi = 0, max_vi = 0, max_ei = 0;
    for (auto& P : plan->parts) {
        sum_vi += P.n_local;
        max_vi = std::max(max_vi, P.n_local);
        max_ei = std::max(max_ei, P.n_edges);
    }
    std::vector<int64_t> inner(p, 0), outer(p, 0);
    for (int i = 0; i < p; ++i)
        for (int j = 0; j < p; ++j) {
            if (i == j) continue;
            int64_t k = (int64_t)mir[i][j].size();
            auto& acc = host[i] == host[j] ? inner : outer;
            acc[i] += k;
            acc[j] += k;
        }
    st.rf = (double)sum_vi / (double)n;
    st.edge_if = (double)max_ei / ((double)m / p);
    st.vertex_if = (double)max_vi / ((double)sum_vi / p);
    st.total_mirrors = sum_vi - n;
    st.inner_max = *std::max_element(inner.begin(), inner.end());
    st.outer_max = *std::max_element(outer.begin(), outer.end());
    st.sum_vi = sum_vi;
    st.max_ei = max_ei;
    if (edge_part_out) std::memcpy(edge_part_out, epart.data(), sizeof(int32_t) * m);
    if (master_out) std::memcpy(master_out, master.data(), sizeof(int32_t) * n);
    *plan_out = plan;
    return CDFGNN_OK;
}

extern "C" int cdfgnn_plan_num_parts(const cdfgnn_plan* plan) { return plan ? plan->p : 0; }

extern "C" int cdfgnn_plan_part(const cdfgnn_plan* plan, int32_t part, cdfgnn_part_view* out) {
    if (!plan || !out) CDF_FAIL(CDFGNN_EUSAGE, "plan/out is NULL");
    if (part < 0 || part >= plan->p) CDF_FAIL(CDFGNN_EUSAGE, "part %d out of range", part);
    const PartData& P = plan->parts[part];
    out->part = part;
    out->n_local = P.n_local;
    out->n_bmaster = P.B;
    out->n_mirror = P.M;
    out->n_edges = P.n_edges;
    out->nnz = (int64_t)P.colidx.size();
    out->local2global = P.l2g.data();
    out->rowptr = P.rowptr.data();
    out->colidx = P.colidx.data();
    out->val = P.val.data();
    out->mirror_off = P.moff.data();
    out->halo_off = P.hoff.data();
    out->halo_local = P.halo_local.data();
    return CDFGNN_OK;
}

extern "C" int cdfgnn_plan_stats(const cdfgnn_plan* plan, cdfgnn_partition_stats* out) {
    if (!plan || !out) CDF_FAIL(CDFGNN_EUSAGE, "plan/out is NULL");
    *out = plan->stats;
    return CDFGNN_OK;
}

extern "C" void cdfgnn_plan_free(cdfgnn_plan* plan) { delete plan; }
