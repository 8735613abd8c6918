// libcdfgnn C ABI: context, workspace carving, halo exchange orchestration,
// layer forward/backward and the Alg. 1 epoch.
//
// Transport (§3.2 gather / scatter): co-resident partitions (world == 1, k == p
// parts on one GPU) and the NVLink push transport (world == p, one part per GPU, peers'
// workspaces mapped with CUDA IPC) use slot-addressed message regions — a message lives in
// the slot of its vertex's halo-list position, stamped with the phase's sequence number, and
// the sending kernel stores it straight into the receiver's region (kernels_halo.cu).  The
// NCCL transport (transport = 1) packs compacted per-peer buffers and exchanges counts and
// payloads with grouped send/recv.  Weight gradients are summed with ncclAllReduce (the
// "parameter server" of P:L221-222, reading R9).
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "common.h"
#include "kernels.h"

namespace cdfgnn {

static thread_local std::string g_err;

void set_error(const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
}

}  // namespace cdfgnn

using namespace cdfgnn;

#define CUDA_TRY(x)                                                                         \
    do {                                                                                    \
        cudaError_t _e = (x);                                                               \
        if (_e != cudaSuccess) CDF_FAIL(CDFGNN_ECUDA, "%s: %s", #x, cudaGetErrorString(_e)); \
    } while (0)
#define NCCL_TRY(x)                                                                         \
    do {                                                                                    \
        ncclResult_t _r = (x);                                                              \
        if (_r != ncclSuccess) CDF_FAIL(CDFGNN_ENCCL, "%s: %s", #x, ncclGetErrorString(_r)); \
    } while (0)

namespace {

struct Bump {
    uint8_t* base = nullptr;
    size_t off = 0;
    template <class T>
    T* take(int64_t count, size_t align = 256) {
        off = (off + align - 1) / align * align;
        T* p = reinterpret_cast<T*>(base + off);
        off += (size_t)std::max<int64_t>(count, 0) * sizeof(T);
        return p;
    }
};

enum Phase { PH_GEMM = 0, PH_SPMM = 1, PH_SYNC = 2, PH_OTHER = 3, PH_END = 4 };
// sub-phases of the halo exchange (tag of PH_SYNC marks)
enum SyncSub { SS_GPACK = 0, SS_GXFER = 1, SS_MASTER = 2, SS_SPACK = 3, SS_SXFER = 4, SS_MIRROR = 5 };

// SpMM work-item schedule of one part for one row-width class (kernels_spmm.cu)
struct SpmmPlan {
    std::vector<int2> items_h, items2_h;   // all rows | [mirror rows][master + interior rows]
    std::vector<int4> split_h;             // per row {partial slot, segments, seg_beg index}
    std::vector<int32_t> seg_beg_h;
    int64_t n_items = 0, n_items_mir = 0, nslots = 0, pstride = 0;
    int2 *items = nullptr, *items2 = nullptr;
    int4* split = nullptr;
    int32_t *seg_beg = nullptr, *pcounter = nullptr;
    float* partial = nullptr;
};

struct LocalPart {
    int32_t part = 0;
    int64_t n = 0, B = 0, M = 0, nnz = 0;
    const int32_t* rowptr_h = nullptr;
    const int32_t* colidx_h = nullptr;
    const float* val_h = nullptr;
    const int32_t* halo_h = nullptr;
    std::vector<int64_t> moff, hoff;
    std::vector<int64_t> capA, capB;   // region capacities per peer
    // device
    int32_t *rowptr = nullptr, *colidx = nullptr, *halo_local = nullptr;
    SpmmPlan sp[2];                    // SpMM work items: [0] wide rows (ld > 64), [1] narrow rows
    float* xT = nullptr;               // cached H^(0)ᵀ (cfg.static_inputs) for ∇W^(0)
    float* hT[CDFGNN_MAX_LAYERS] = {}; // H^(l)ᵀ written with the forward ReLU (epoch, tcgen05 path)
    const float* hT_src[CDFGNN_MAX_LAYERS] = {};   // the H^(l) buffer hT[l] mirrors
    const float* xT_src = nullptr;     // the X pointer xT was built from
    float* ax = nullptr;               // cfg.static_inputs == 2: Â_i X_i, built once per X pointer
    const float* ax_src = nullptr;     // (xT then holds (Â_i X_i)ᵀ)
    float* val = nullptr;
    int64_t *moff_d = nullptr, *hoff_d = nullptr;
    uint8_t* regA[kMaxParts] = {};
    uint8_t* regB[kMaxParts] = {};
    RegionTab *gsend_d = nullptr, *grecv_d = nullptr, *ssend_d = nullptr, *srecv_d = nullptr;
    RegionTab gsend_h{}, grecv_h{}, ssend_h{}, srecv_h{};
    PutTab *putG_d = nullptr, *putS_d = nullptr;   // NVLink push of gather / scatter messages
    SlotTab gdst{}, gsrc{}, sdst{}, ssrc{};   // slot layout: gather / scatter destination and source regions
    int32_t* hpos = nullptr;           // [B*p] slot of master row r in the halo list shared with part s
    std::vector<int32_t> hpos_h;
    uint64_t* bar = nullptr;           // [p] NVLink barrier arrival slots (written by the peers)
    int32_t* cnt = nullptr;           // [4p]: gsend | grecv | ssend | srecv
    int32_t* cnt_h = nullptr;         // pinned
    uint8_t *gflag = nullptr, *fired = nullptr, *active = nullptr;   // [L][2][M] / [L][2][B] per sync
    int32_t *idxmap = nullptr, *mmap = nullptr;
    uint8_t* stage_codes = nullptr;
    float *stage_lohi = nullptr, *stage_a = nullptr;
    CacheDev cache[CDFGNN_MAX_LAYERS][2] = {};
    float* act[CDFGNN_MAX_LAYERS + 1] = {};
    float *T = nullptr, *S = nullptr, *D[2] = {nullptr, nullptr}, *rowloss = nullptr;
    float* X_stage = nullptr;          // host-input staging, slot 0 ...
    int32_t* lab_stage = nullptr;
    uint8_t* mask_stage = nullptr;
    float* X_stage1 = nullptr;         // ... and slot 1 (prefetch of the next step's inputs)
    float* xpack = nullptr;            // world > 1: master rows of X packed per mirror peer
    int32_t* lab_stage1 = nullptr;
    uint8_t* mask_stage1 = nullptr;
    HaloDev halo{};
};

}  // namespace

struct cdfgnn_ctx {
    cdfgnn_cfg cfg{};
    int32_t p = 0, k = 0, rank = 0, world = 1, device = 0;
    std::vector<LocalPart> parts;
    ncclComm_t comm = nullptr;
    int64_t Fmax = 0, ldmax = 0, hdr_bytes = 4, wtotal = 0, rowb_max = 0;
    bool slot = false;                 // slot-addressed message layout (co-resident, NVLink push)
    uint32_t seq = 0;                  // message stamps (slot layout), identical on every rank
    uint32_t stamp[CDFGNN_MAX_LAYERS][2][2] = {};   // (l, dir) -> gather / scatter stamp of the sync in flight
    uint32_t last_stamp[2] = {0, 0};   // most recent gather / scatter stamp (cdfgnn_msg_view)
    int64_t last_ld[2] = {0, 0};
    int64_t woff[CDFGNN_MAX_LAYERS + 1] = {};
    int64_t splitk_cap = 0;
    float *dW = nullptr, *adam_m = nullptr, *adam_v = nullptr, *splitk = nullptr;
    float* wpad = nullptr;             // W^(l) with zero-padded rows of ld(F_l) (TMA strides)
    int64_t wpoff[CDFGNN_MAX_LAYERS + 1] = {};
    float* wtpad = nullptr;            // W^(l)ᵀ [F_l x ld(F_{l-1})] (K-major B of T = H W)
    int64_t wtoff[CDFGNN_MAX_LAYERS + 1] = {};
    float *trA = nullptr, *trB = nullptr;   // K-major copies Hᵀ, Sᵀ for ∇W (tcgen05 path)
    int64_t npad = 0, fin_max = 0;
    unsigned long long* stats_d = nullptr;    // [L][2][4]
    unsigned long long* stats_h = nullptr;    // pinned
    double* loss_d = nullptr;        // [k]
    double* loss_part = nullptr;     // [148] partial sums of the row losses
    int32_t* scal_d = nullptr;       // [0] correct, [1] err, [2] ntrain
    double* host_scratch = nullptr;  // pinned: k doubles + ints
    int64_t ntrain = -1;
    double eps = 0.01, mean_acc = 0.0;
    bool have_mean = false;
    int64_t step_t = 0;
    int launches = 0;
    bool timing = false;
    std::vector<cudaEvent_t> ev;
    std::vector<int> ev_phase;
    std::vector<int64_t> ev_tag;   // SpMM: row width ld of the launch
    size_t ev_used = 0;
    size_t ws_bytes = 0;
    void* ws = nullptr;
    int transport = 0;                 // 0 co-resident (world 1), 1 NCCL send/recv, 2 NVLink push
    bool in_epoch = false;             // Hᵀ reuse between forward and backward only inside cdfgnn_epoch
    std::vector<void*> peer_maps;      // IPC-opened peer allocations (push transport)
    BarTab bar{};                      // device barrier over the mappings (push transport)
    uint64_t bar_seq = 0;
    bool bar_dev = false;              // false: NCCL allreduce barrier (CDFGNN_NCCL_BARRIER=1)
    // boundary-rows-first overlap (cfg.overlap): gather phases run on s2
    cudaStream_t s2 = nullptr;
    cudaEvent_t evA = nullptr, evB = nullptr;
    bool pend[CDFGNN_MAX_LAYERS][2] = {};   // gather of (l, dir) already launched on s2
    // pipelined host inputs (cdfgnn_epoch_host_next): staging slot prefetched for the next call
    cudaStream_t cs = nullptr;
    cudaEvent_t staged[2] = {nullptr, nullptr}, used[2] = {nullptr, nullptr};
    int prefetched = -1;
    // world > 1: input rows of mirrors are filled from their masters over NCCL (own communicator,
    // issued only on the copy stream cs), so each vertex's features cross PCIe once
    ncclComm_t comm_in = nullptr;
    // §8 f2: each layer's ∇W allreduce runs on its own communicator and stream as soon as the
    // layer's ∇W is complete, under the lower layers' backward (reading R8); joined before the
    // optimizer
    ncclComm_t comm_grad = nullptr;
    cudaStream_t s3 = nullptr;
    cudaEvent_t evG = nullptr, evJ = nullptr;
    bool dw_pending = false;
    bool relu_z = false;               // the sync in flight writes σ(Z) (fused ReLU, fwd_impl)
};

namespace {

int64_t sync_width(const cdfgnn_ctx* c, int l) { return c->cfg.dims[l]; }

// SpMM work items of a part (kernels_spmm.cu).  phases > 1: rows with more than
// `min_deg` neighbours are split by column range into `phases` segments, visited
// phase-major (each segment list longest first), then the unsplit rows longest first.
// Else chunk > 0: rows longer than `chunk` neighbours become ceil(deg/chunk) chunks and
// every item is visited longest first.  items2_h holds the same items with the mirror
// rows' first (boundary-rows-first scheduling, §8 f1), order otherwise kept.
int env_knob(const char* name, int dflt) {
    const char* e = getenv(name);    // tuning knobs for tools/spmm_bench.py
    return e ? atoi(e) : dflt;
}

void build_spmm_items(const LocalPart& P, SpmmPlan& S, int chunk, int phases, int min_deg) {
    S.split_h.assign(P.n, make_int4(-1, 0, 0, 0));
    S.seg_beg_h.clear();
    S.nslots = 0;
    std::vector<std::pair<int32_t, int2>> w;      // (weight, item)
    std::vector<std::pair<int32_t, int2>> tail;   // unsplit rows (phase mode)
    w.reserve(P.n);
    auto split_row = [&](int64_t r, const std::vector<int32_t>& starts) {
        const int nseg = (int)starts.size() - 1;
        S.split_h[r] = make_int4((int)S.nslots, nseg, (int)S.seg_beg_h.size(), 0);
        S.nslots += nseg;
        S.seg_beg_h.insert(S.seg_beg_h.end(), starts.begin(), starts.end());
    };
    if (phases > 1) {
        std::vector<std::vector<std::pair<int32_t, int2>>> ph(phases);
        std::vector<int32_t> st(phases + 1);
        for (int64_t r = 0; r < P.n; ++r) {
            const int32_t rb = P.rowptr_h[r], re = P.rowptr_h[r + 1];
            if (re - rb <= min_deg) {
                tail.push_back({re - rb, make_int2((int)r, -1)});
                continue;
            }
            st[0] = rb;
            st[phases] = re;
            for (int k = 1; k < phases; ++k) {
                const int32_t bound = (int32_t)((int64_t)k * P.n / phases);
                st[k] = (int32_t)(std::lower_bound(P.colidx_h + rb, P.colidx_h + re, bound) - P.colidx_h);
            }
            split_row(r, st);
            for (int k = 0; k < phases; ++k) ph[k].push_back({st[k + 1] - st[k], make_int2((int)r, k)});
        }
        auto by_weight = [](const std::pair<int32_t, int2>& a, const std::pair<int32_t, int2>& b) {
            return a.first > b.first;
        };
        for (auto& v : ph) {
            std::stable_sort(v.begin(), v.end(), by_weight);
            w.insert(w.end(), v.begin(), v.end());
        }
        std::stable_sort(tail.begin(), tail.end(), by_weight);
        w.insert(w.end(), tail.begin(), tail.end());
    } else {
        std::vector<int32_t> st;
        for (int64_t r = 0; r < P.n; ++r) {
            const int32_t rb = P.rowptr_h[r], re = P.rowptr_h[r + 1], deg = re - rb;
            if (chunk > 0 && deg > chunk) {
                const int32_t nch = (deg + chunk - 1) / chunk;
                st.resize(nch + 1);
                for (int32_t ch = 0; ch < nch; ++ch) st[ch] = rb + ch * chunk;
                st[nch] = re;
                split_row(r, st);
                for (int32_t ch = 0; ch < nch; ++ch)
                    w.push_back({std::min(chunk, deg - ch * chunk), make_int2((int)r, ch)});
            } else {
                w.push_back({deg, make_int2((int)r, -1)});
            }
        }
        // order: 0 = longest first (LPT); 1 = row order (locality of the local numbering);
        // 2 = items longer than CDFGNN_SPMM_HEAVY neighbours longest first, then row order
        const int order = env_knob("CDFGNN_SPMM_ORDER", 0);
        auto by_weight = [](const std::pair<int32_t, int2>& a, const std::pair<int32_t, int2>& b) {
            return a.first > b.first;
        };
        if (order == 0) {
            std::stable_sort(w.begin(), w.end(), by_weight);
        } else if (order == 2) {
            const int32_t heavy = env_knob("CDFGNN_SPMM_HEAVY", 4096);
            auto mid = std::stable_partition(w.begin(), w.end(),
                                             [&](const std::pair<int32_t, int2>& a) { return a.first > heavy; });
            std::stable_sort(w.begin(), mid, by_weight);
        }
    }
    if (S.seg_beg_h.empty()) S.seg_beg_h.push_back(0);
    S.n_items = (int64_t)w.size();
    S.items_h.resize(w.size());
    for (size_t i = 0; i < w.size(); ++i) S.items_h[i] = w[i].second;
    S.items2_h.clear();
    S.items2_h.reserve(w.size());
    auto is_mirror = [&](const int2& it) { return it.x >= P.B && it.x < P.B + P.M; };
    for (const int2& it : S.items_h)
        if (is_mirror(it)) S.items2_h.push_back(it);
    S.n_items_mir = (int64_t)S.items2_h.size();
    for (const int2& it : S.items_h)
        if (!is_mirror(it)) S.items2_h.push_back(it);
}

SpmmPlan& spmm_plan(LocalPart& P, int64_t ld) { return P.sp[ld <= 64 ? 1 : 0]; }

SpmmItems spmm_items(LocalPart& P, int rows, int64_t ld) {
    const SpmmPlan& S = spmm_plan(P, ld);
    SpmmItems it;
    it.items = rows == 0 ? S.items : (rows == 1 ? S.items2 : S.items2 + S.n_items_mir);
    it.split = S.split;
    it.seg_beg = S.seg_beg;
    it.partial = S.partial;
    it.counter = S.pcounter;
    return it;
}

// host-side sizes from the plan
int prepare(cdfgnn_ctx* c, const cdfgnn_plan* plan, const int32_t* parts, int32_t k,
            const cdfgnn_cfg* cfg) {
    if (!plan || !cfg) CDF_FAIL(CDFGNN_EUSAGE, "plan/cfg is NULL");
    c->cfg = *cfg;
    c->p = cdfgnn_plan_num_parts(plan);
    c->k = k;
    if (cfg->L < 1 || cfg->L > CDFGNN_MAX_LAYERS) CDF_FAIL(CDFGNN_EUSAGE, "L must be in [1, %d]", CDFGNN_MAX_LAYERS);
    if (cfg->quant_bits != 0 && cfg->quant_bits != 4 && cfg->quant_bits != 8 && cfg->quant_bits != 16)
        CDF_FAIL(CDFGNN_EUSAGE, "quant_bits must be 0, 4, 8 or 16");
    if (cfg->msg_layout < 0 || cfg->msg_layout > 2) CDF_FAIL(CDFGNN_EUSAGE, "msg_layout must be 0, 1 or 2");
    for (int l = 0; l <= cfg->L; ++l)
        if (cfg->dims[l] < 1) CDF_FAIL(CDFGNN_EUSAGE, "dims[%d] must be >= 1", l);
    for (int l = 1; l <= cfg->L; ++l)
        if (cfg->dims[l] > 1024) CDF_FAIL(CDFGNN_EUSAGE, "hidden/output widths must be <= 1024");
    if (cfg->dims[cfg->L] > 256) CDF_FAIL(CDFGNN_EUSAGE, "at most 256 classes");
    if (k < 1 || k > c->p) CDF_FAIL(CDFGNN_EUSAGE, "k must be in [1, p]");
    c->Fmax = 0;
    for (int l = 1; l <= cfg->L; ++l) c->Fmax = std::max<int64_t>(c->Fmax, cfg->dims[l]);
    c->ldmax = ld_of(c->Fmax);
    c->hdr_bytes = cfg->quant_bits ? 12 : 4;
    c->rowb_max = code_row_bytes(cfg->quant_bits, c->ldmax);
    c->wtotal = 0;
    for (int l = 1; l <= cfg->L; ++l) {
        c->woff[l - 1] = c->wtotal;
        c->wtotal += (int64_t)cfg->dims[l - 1] * cfg->dims[l];
    }
    c->woff[cfg->L] = c->wtotal;
    int64_t wp = 0;
    for (int l = 1; l <= cfg->L; ++l) {
        c->wpoff[l - 1] = wp;
        wp += align_up((int64_t)cfg->dims[l - 1] * ld_of(cfg->dims[l]), 64);
    }
    c->wpoff[cfg->L] = wp;
    int64_t wt = 0;
    for (int l = 1; l <= cfg->L; ++l) {
        c->wtoff[l - 1] = wt;
        wt += align_up((int64_t)cfg->dims[l] * ld_of(cfg->dims[l - 1]), 64);
        c->fin_max = std::max<int64_t>(c->fin_max, cfg->dims[l - 1]);
    }
    c->wtoff[cfg->L] = wt;
    int64_t maxw = 0;
    for (int l = 1; l <= cfg->L; ++l) maxw = std::max<int64_t>(maxw, (int64_t)cfg->dims[l - 1] * cfg->dims[l]);
    c->splitk_cap = 64 * maxw;
    if (c->cfg.static_inputs < 0 || c->cfg.static_inputs > 2) CDF_FAIL(CDFGNN_EUSAGE, "static_inputs must be 0, 1 or 2");
    c->parts.assign(k, LocalPart());
    for (int t = 0; t < k; ++t) {
        cdfgnn_part_view v;
        CDF_TRY(cdfgnn_plan_part(plan, parts[t], &v));
        LocalPart& P = c->parts[t];
        P.part = parts[t];
        P.n = v.n_local; P.B = v.n_bmaster; P.M = v.n_mirror; P.nnz = v.nnz;
        P.rowptr_h = v.rowptr; P.colidx_h = v.colidx; P.val_h = v.val; P.halo_h = v.halo_local;
        P.moff.assign(v.mirror_off, v.mirror_off + c->p + 1);
        P.hoff.assign(v.halo_off, v.halo_off + c->p + 1);
        P.capA.resize(c->p); P.capB.resize(c->p);
        for (int j = 0; j < c->p; ++j) {
            P.capA[j] = P.moff[j + 1] - P.moff[j];
            P.capB[j] = P.hoff[j + 1] - P.hoff[j];
        }
        // slot of each boundary master row in the halo list shared with each peer (static)
        P.hpos_h.assign((size_t)P.B * c->p, -1);
        for (int q = 0; q < c->p; ++q)
            for (int64_t k = P.hoff[q]; k < P.hoff[q + 1]; ++k)
                P.hpos_h[(size_t)v.halo_local[k] * c->p + q] = (int32_t)(k - P.hoff[q]);
        // wide rows: LPT over whole rows (chunks cost L2 bandwidth there, profiles/r1);
        // narrow rows: hub rows split into chunks (their latency chains dominated)
        build_spmm_items(P, P.sp[0], spmm_chunk(true, P.nnz), spmm_default_phases(), spmm_phase_min_degree());
        build_spmm_items(P, P.sp[1], spmm_chunk(false, P.nnz), spmm_default_phases(), spmm_phase_min_degree());
        P.sp[0].pstride = c->ldmax;
        P.sp[1].pstride = std::min<int64_t>(c->ldmax, 64);
    }
    return CDFGNN_OK;
}

// a region holds either layout: compacted (header array, then rows) or slot-addressed
int64_t region_bytes(const cdfgnn_ctx* c, int64_t cap) {
    const int64_t packed = align_up(cap * c->hdr_bytes, 256) + cap * c->rowb_max;
    return std::max(packed, cap * slot_stride(c->cfg.quant_bits, c->ldmax));
}

void carve(cdfgnn_ctx* c, Bump& b) {
    const int p = c->p, L = c->cfg.L;
    for (LocalPart& P : c->parts) {
        P.rowptr = b.take<int32_t>(P.n + 1);
        P.colidx = b.take<int32_t>(P.nnz);
        for (SpmmPlan& S : P.sp) {
            S.items = b.take<int2>(S.n_items);
            S.items2 = b.take<int2>(S.n_items);
            S.split = b.take<int4>(P.n);
            S.seg_beg = b.take<int32_t>((int64_t)S.seg_beg_h.size());
            S.pcounter = b.take<int32_t>(S.nslots);
            S.partial = b.take<float>(S.nslots * S.pstride);
        }
        P.val = b.take<float>(P.nnz);
        P.halo_local = b.take<int32_t>(P.hoff[p]);
        P.moff_d = b.take<int64_t>(p + 1);
        P.hoff_d = b.take<int64_t>(p + 1);
        for (int j = 0; j < p; ++j) {
            P.regA[j] = b.take<uint8_t>(region_bytes(c, P.capA[j]));
            P.regB[j] = b.take<uint8_t>(region_bytes(c, P.capB[j]));
        }
        P.gsend_d = b.take<RegionTab>(1);
        P.grecv_d = b.take<RegionTab>(1);
        P.ssend_d = b.take<RegionTab>(1);
        P.srecv_d = b.take<RegionTab>(1);
        P.putG_d = b.take<PutTab>(1);
        P.putS_d = b.take<PutTab>(1);
        P.cnt = b.take<int32_t>(4 * p);
        P.bar = b.take<uint64_t>(p);
        P.gflag = b.take<uint8_t>(2 * L * P.M);
        P.fired = b.take<uint8_t>(2 * L * P.B);
        P.active = b.take<uint8_t>(2 * L * P.B);
        P.hpos = b.take<int32_t>((int64_t)p * P.B);
        P.idxmap = b.take<int32_t>((int64_t)p * P.B);
        P.mmap = b.take<int32_t>(P.M);
        P.stage_codes = b.take<uint8_t>(P.B * c->rowb_max);
        P.stage_lohi = b.take<float>(2 * P.B);
        P.stage_a = b.take<float>(P.B * c->ldmax);
        for (int l = 1; l <= L; ++l) {
            const int64_t ld = ld_of(c->cfg.dims[l]);
            for (int dir = 0; dir < 2; ++dir) {
                CacheDev& cd = P.cache[l - 1][dir];
                if (c->cfg.cache_on) {
                    cd.s_mir = b.take<float>(P.M * ld);
                    cd.b_mir = b.take<float>(P.M * ld);
                    cd.s_mas = b.take<float>(P.B * ld);
                    cd.a = b.take<float>(P.B * ld);
                    cd.b_mas = b.take<float>(P.B * ld);
                } else {
                    cd = CacheDev{};
                }
            }
            P.act[l] = b.take<float>(P.n * ld);
        }
        P.T = b.take<float>(P.n * c->ldmax);
        P.S = b.take<float>(P.n * c->ldmax);
        P.D[0] = b.take<float>(P.n * c->ldmax);
        P.D[1] = b.take<float>(P.n * c->ldmax);
        P.rowloss = b.take<float>(P.n);
        P.X_stage = b.take<float>(P.n * ld_of(c->cfg.dims[0]));
        if (c->cfg.static_inputs == 2) P.ax = b.take<float>(P.n * ld_of(c->cfg.dims[0]));
        P.lab_stage = b.take<int32_t>(P.n);
        P.mask_stage = b.take<uint8_t>(P.n);
        P.X_stage1 = b.take<float>(P.n * ld_of(c->cfg.dims[0]));
        if (c->k == 1 && p > 1) P.xpack = b.take<float>(P.hoff[p] * ld_of(c->cfg.dims[0]));   // one part per rank
        P.lab_stage1 = b.take<int32_t>(P.n);
        P.mask_stage1 = b.take<uint8_t>(P.n);
    }
    c->dW = b.take<float>(c->wtotal);
    c->adam_m = b.take<float>(c->wtotal);
    c->adam_v = b.take<float>(c->wtotal);
    c->splitk = b.take<float>(c->splitk_cap);
    c->wpad = b.take<float>(c->wpoff[c->cfg.L]);
    c->wtpad = b.take<float>(c->wtoff[c->cfg.L]);
    int64_t nmax = 0;
    for (const LocalPart& P : c->parts) nmax = std::max(nmax, P.n);
    c->npad = ld_of(nmax);
    if (c->cfg.gemm_tf32) {
        c->trA = b.take<float>(c->fin_max * c->npad);
        c->trB = b.take<float>(c->Fmax * c->npad);
        if (c->cfg.static_inputs)
            for (LocalPart& P : c->parts) P.xT = b.take<float>((int64_t)c->cfg.dims[0] * ld_of(P.n));
        for (LocalPart& P : c->parts)
            for (int l = 1; l < c->cfg.L; ++l) P.hT[l] = b.take<float>((int64_t)c->cfg.dims[l] * ld_of(P.n));
    }
    c->stats_d = b.take<unsigned long long>(CDFGNN_MAX_LAYERS * 2 * 4);
    c->loss_d = b.take<double>(std::max(c->k, 1));
    c->loss_part = b.take<double>(148);
    c->scal_d = b.take<int32_t>(8);
}

// ---- phase timing ----------------------------------------------------------------
void mark(cdfgnn_ctx* c, int phase, cudaStream_t s, int64_t tag = 0) {
    // phase times are reported per cdfgnn_epoch (the event list restarts with every epoch)
    if (!c->timing || !c->in_epoch) return;
    if (c->ev_used >= c->ev.size()) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) return;
        c->ev.push_back(e);
        c->ev_phase.push_back(0);
        c->ev_tag.push_back(0);
    }
    cudaEventRecord(c->ev[c->ev_used], s);
    c->ev_phase[c->ev_used] = phase;
    c->ev_tag[c->ev_used] = tag;
    c->ev_used++;
}

void build_tables(cdfgnn_ctx* c) {
    const int p = c->p;
    for (int t = 0; t < c->k; ++t) {
        LocalPart& P = c->parts[t];
        int32_t* cg_send = P.cnt;
        int32_t* cg_recv = P.cnt + p;
        int32_t* cs_send = P.cnt + 2 * p;
        int32_t* cs_recv = P.cnt + 3 * p;
        for (int j = 0; j < p; ++j) {
            P.gsend_h.hdr[j] = P.regA[j];
            P.gsend_h.pay[j] = P.regA[j] + align_up(P.capA[j] * c->hdr_bytes, 256);
            P.gsend_h.cnt[j] = cg_send + j;
            P.ssend_h.hdr[j] = P.regB[j];
            P.ssend_h.pay[j] = P.regB[j] + align_up(P.capB[j] * c->hdr_bytes, 256);
            P.ssend_h.cnt[j] = cs_send + j;
        }
    }
    for (int t = 0; t < c->k; ++t) {
        LocalPart& P = c->parts[t];
        const int me = P.part;
        for (int s = 0; s < p; ++s) {
            if (c->world == 1) {
                // co-resident partitions: read the sender's region in place
                LocalPart& Q = c->parts[s];
                // slot layout: a sender stores into its own region, the receiver reads it there
                P.gdst.base[s] = s == me ? nullptr : P.regA[s];
                P.gsrc.base[s] = s == me ? nullptr : Q.regA[me];
                P.sdst.base[s] = s == me ? nullptr : P.regB[s];
                P.ssrc.base[s] = s == me ? nullptr : Q.regB[me];
                P.grecv_h.hdr[s] = Q.gsend_h.hdr[me];
                P.grecv_h.pay[s] = Q.gsend_h.pay[me];
                P.grecv_h.cnt[s] = Q.gsend_h.cnt[me];
                P.srecv_h.hdr[s] = Q.ssend_h.hdr[me];
                P.srecv_h.pay[s] = Q.ssend_h.pay[me];
                P.srecv_h.cnt[s] = Q.ssend_h.cnt[me];
            } else {
                P.grecv_h.hdr[s] = P.regB[s];
                P.grecv_h.pay[s] = P.ssend_h.pay[s];
                P.grecv_h.cnt[s] = P.cnt + p + s;
                P.srecv_h.hdr[s] = P.regA[s];
                P.srecv_h.pay[s] = P.gsend_h.pay[s];
                P.srecv_h.cnt[s] = P.cnt + 3 * p + s;
                // slot layout (push): receive in the own regions; destinations are mapped by
                // setup_push (peers' regB[me] for the gather, regA[me] for the scatter)
                P.gsrc.base[s] = s == me ? nullptr : P.regB[s];
                P.ssrc.base[s] = s == me ? nullptr : P.regA[s];
            }
        }
        HaloDev& h = P.halo;
        h.me = me; h.p = p; h.n = P.n; h.B = P.B; h.M = P.M;
        h.quant = c->cfg.quant_bits; h.hdr_bytes = c->hdr_bytes;
        h.moff = P.moff_d; h.hoff = P.hoff_d; h.halo_local = P.halo_local;
        h.gsend = P.gsend_d; h.grecv = P.grecv_d; h.ssend = P.ssend_d; h.srecv = P.srecv_d;
        h.remote = 0;
        h.gflag = P.gflag; h.fired = P.fired; h.active = P.active;
        h.idxmap = P.idxmap; h.mmap = P.mmap;
        h.stage_codes = P.stage_codes; h.stage_lohi = P.stage_lohi; h.stage_a = P.stage_a;
        h.err = c->scal_d + 1;
        h.hpos = P.hpos;
    }
}

// CDFGNN_DEBUG_SYNC=1: synchronise after every launch group to localise faults
bool debug_sync() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("CDFGNN_DEBUG_SYNC");
        v = (e && e[0] == '1') ? 1 : 0;
    }
    return v == 1;
}

int check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess && debug_sync()) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) CDF_FAIL(CDFGNN_ECUDA, "%s: %s", what, cudaGetErrorString(e));
    return CDFGNN_OK;
}

// Host wait on `s` that notices a failed or dead peer: while the stream is busy, poll the
// communicators' asynchronous error state; an NCCL error aborts the communicators (so
// their kernels return) and maps to ENCCL instead of hanging in cudaStreamSynchronize.
int wait_stream(cdfgnn_ctx* c, cudaStream_t s) {
    if (!c->comm) {
        CUDA_TRY(cudaStreamSynchronize(s));
        return CDFGNN_OK;
    }
    for (unsigned spin = 0;; ++spin) {
        const cudaError_t e = cudaStreamQuery(s);
        if (e == cudaSuccess) return CDFGNN_OK;
        if (e != cudaErrorNotReady) CDF_FAIL(CDFGNN_ECUDA, "stream: %s", cudaGetErrorString(e));
        for (ncclComm_t cm : {c->comm, c->comm_in, c->comm_grad}) {
            if (!cm) continue;
            ncclResult_t ae = ncclSuccess;
            if (ncclCommGetAsyncError(cm, &ae) == ncclSuccess && ae != ncclSuccess && ae != ncclInProgress) {
                ncclCommAbort(c->comm);
                if (c->comm_in) ncclCommAbort(c->comm_in);
                if (c->comm_grad) ncclCommAbort(c->comm_grad);
                c->comm = c->comm_in = c->comm_grad = nullptr;
                CDF_FAIL(CDFGNN_ENCCL, "NCCL asynchronous error: %s", ncclGetErrorString(ae));
            }
        }
        if (spin > 64) std::this_thread::yield();
    }
}

// NCCL count + payload exchange for one phase (world > 1, k == 1)
int nccl_phase(cdfgnn_ctx* c, LocalPart& P, bool gather, int64_t rowb, cudaStream_t s,
               int64_t* wire) {
    const int p = c->p, me = P.part;
    int32_t* snd = gather ? P.cnt : P.cnt + 2 * p;
    int32_t* rcv = gather ? P.cnt + p : P.cnt + 3 * p;
    NCCL_TRY(ncclGroupStart());
    for (int j = 0; j < p; ++j) {
        if (j == me) continue;
        NCCL_TRY(ncclSend(snd + j, 1, ncclInt32, j, c->comm, s));
        NCCL_TRY(ncclRecv(rcv + j, 1, ncclInt32, j, c->comm, s));
    }
    NCCL_TRY(ncclGroupEnd());
    CUDA_TRY(cudaMemcpyAsync(P.cnt_h, P.cnt, sizeof(int32_t) * 4 * p, cudaMemcpyDeviceToHost, s));
    CDF_TRY(wait_stream(c, s));
    const int32_t* hs = P.cnt_h + (gather ? 0 : 2 * p);
    const int32_t* hr = P.cnt_h + (gather ? p : 3 * p);
    const RegionTab& st = gather ? P.gsend_h : P.ssend_h;
    const RegionTab& rt = gather ? P.grecv_h : P.srecv_h;
    const std::vector<int64_t>& scap = gather ? P.capA : P.capB;
    const std::vector<int64_t>& rcap = gather ? P.capB : P.capA;
    for (int j = 0; j < p; ++j) {
        if (j == me) continue;
        if (hs[j] < 0 || hs[j] > scap[j] || hr[j] < 0 || hr[j] > rcap[j])
            CDF_FAIL(CDFGNN_EPROTO, "message count out of range (peer %d: send %d/%lld recv %d/%lld)",
                     j, hs[j], (long long)scap[j], hr[j], (long long)rcap[j]);
    }
    NCCL_TRY(ncclGroupStart());
    for (int j = 0; j < p; ++j) {
        if (j == me) continue;
        if (hs[j] > 0) {
            NCCL_TRY(ncclSend(st.hdr[j], (size_t)hs[j] * c->hdr_bytes, ncclUint8, j, c->comm, s));
            NCCL_TRY(ncclSend(st.pay[j], (size_t)hs[j] * rowb, ncclUint8, j, c->comm, s));
            *wire += (int64_t)hs[j] * (c->hdr_bytes + rowb);
        }
        if (hr[j] > 0) {
            NCCL_TRY(ncclRecv(rt.hdr[j], (size_t)hr[j] * c->hdr_bytes, ncclUint8, j, c->comm, s));
            NCCL_TRY(ncclRecv(rt.pay[j], (size_t)hr[j] * rowb, ncclUint8, j, c->comm, s));
        }
    }
    NCCL_TRY(ncclGroupEnd());
    return CDFGNN_OK;
}

// NVLink push: every rank's pack kernels have stored into the peers' receive regions once
// this stream-ordered all-reduce completes on all ranks (no host round trip)
int push_barrier(cdfgnn_ctx* c, cudaStream_t s) {
    if (c->bar_dev) {
        c->launches += launch_nvl_barrier(c->bar, ++c->bar_seq, c->scal_d + 1, s);
        return check_launch("nvl barrier");
    }
    NCCL_TRY(ncclAllReduce(c->scal_d + 4, c->scal_d + 4, 1, ncclInt32, ncclSum, c->comm, s));
    return CDFGNN_OK;
}

struct PeerInfo {
    cudaIpcMemHandle_t handle;
    uint64_t ws_off;                   // workspace offset inside the IPC allocation
    uint64_t cnt_off;                  // counts array, relative to the workspace
    uint64_t bar_off;                  // barrier arrival slots, relative to the workspace
    uint64_t regA_off[kMaxParts];      // mirror-role regions (receive scatter from master j)
    uint64_t regB_off[kMaxParts];      // master-role regions (receive gather from source s)
};

typedef CUresult (*GetRangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);

// Map every peer's receive regions into this process (CUDA IPC over NVLink) and point
// the send tables at them.  Returns non-OK (caller falls back to NCCL) if IPC fails.
int setup_push(cdfgnn_ctx* c, cudaStream_t s) {
    void* fnp = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fnp, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
        CDF_FAIL(CDFGNN_ECUDA, "cuMemGetAddressRange unavailable");
    CUdeviceptr base = 0;
    size_t sz = 0;
    if (reinterpret_cast<GetRangeFn>(fnp)(&base, &sz, (CUdeviceptr)c->ws) != CUDA_SUCCESS)
        CDF_FAIL(CDFGNN_ECUDA, "cuMemGetAddressRange failed");
    LocalPart& P = c->parts[0];
    const int p = c->p, me = P.part;
    PeerInfo mine;
    std::memset(&mine, 0, sizeof(mine));
    if (cudaIpcGetMemHandle(&mine.handle, (void*)base) != cudaSuccess) {
        cudaGetLastError();
        CDF_FAIL(CDFGNN_ECUDA, "cudaIpcGetMemHandle failed (workspace not IPC-shareable)");
    }
    const uint8_t* ws = reinterpret_cast<const uint8_t*>(c->ws);
    mine.ws_off = (uint64_t)(ws - reinterpret_cast<const uint8_t*>(base));
    mine.cnt_off = (uint64_t)(reinterpret_cast<const uint8_t*>(P.cnt) - ws);
    mine.bar_off = (uint64_t)(reinterpret_cast<const uint8_t*>(P.bar) - ws);
    for (int j = 0; j < p; ++j) {
        mine.regA_off[j] = (uint64_t)(P.regA[j] - ws);
        mine.regB_off[j] = (uint64_t)(P.regB[j] - ws);
    }
    // all-gather the tables through NCCL (device staging in the split-K scratch)
    uint8_t* dsend = reinterpret_cast<uint8_t*>(c->splitk);
    uint8_t* drecv = dsend + align_up(sizeof(PeerInfo), 256);
    if ((int64_t)(align_up(sizeof(PeerInfo), 256) + sizeof(PeerInfo) * p) > c->splitk_cap * 4)
        CDF_FAIL(CDFGNN_EUSAGE, "scratch too small for the peer table");
    std::vector<PeerInfo> all(p);
    CUDA_TRY(cudaMemcpyAsync(dsend, &mine, sizeof(mine), cudaMemcpyHostToDevice, s));
    NCCL_TRY(ncclAllGather(dsend, drecv, sizeof(PeerInfo), ncclUint8, c->comm, s));
    CUDA_TRY(cudaMemcpyAsync(all.data(), drecv, sizeof(PeerInfo) * p, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    PutTab pg, ps;
    std::memset(&pg, 0, sizeof(pg));
    std::memset(&ps, 0, sizeof(ps));
    for (int r = 0; r < p; ++r) {
        if (r == me) continue;
        void* mapped = nullptr;
        if (cudaIpcOpenMemHandle(&mapped, all[r].handle, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
            cudaGetLastError();
            for (void* m : c->peer_maps) cudaIpcCloseMemHandle(m);
            c->peer_maps.clear();
            CDF_FAIL(CDFGNN_ECUDA, "cudaIpcOpenMemHandle failed for peer %d", r);
        }
        c->peer_maps.push_back(mapped);
        uint8_t* pws = reinterpret_cast<uint8_t*>(mapped) + all[r].ws_off;
        c->bar.peer_slot[r] = reinterpret_cast<uint64_t*>(pws + all[r].bar_off) + me;
        int32_t* pcnt = reinterpret_cast<int32_t*>(pws + all[r].cnt_off);
        // gather: my packed mirror slab for master r -> r's master-role region for source me
        pg.src_hdr[r] = P.gsend_h.hdr[r];
        pg.src_pay[r] = P.gsend_h.pay[r];
        pg.src_cnt[r] = P.gsend_h.cnt[r];
        pg.dst_hdr[r] = pws + all[r].regB_off[me];
        pg.dst_pay[r] = pg.dst_hdr[r] + align_up(P.capA[r] * c->hdr_bytes, 256);
        pg.dst_cnt[r] = pcnt + p + me;
        // scatter: my packed halo list for mirror part r -> r's mirror-role region for master me
        ps.src_hdr[r] = P.ssend_h.hdr[r];
        ps.src_pay[r] = P.ssend_h.pay[r];
        ps.src_cnt[r] = P.ssend_h.cnt[r];
        ps.dst_hdr[r] = pws + all[r].regA_off[me];
        ps.dst_pay[r] = ps.dst_hdr[r] + align_up(P.capB[r] * c->hdr_bytes, 256);
        ps.dst_cnt[r] = pcnt + 3 * p + me;
        // slot layout: the kernels store straight into the peer's regions
        P.gdst.base[r] = pg.dst_hdr[r];
        P.sdst.base[r] = ps.dst_hdr[r];
    }
    CUDA_TRY(cudaMemcpyAsync(P.putG_d, &pg, sizeof(PutTab), cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(P.putS_d, &ps, sizeof(PutTab), cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    c->bar.my_slots = P.bar;
    c->bar.p = p;
    c->bar.me = me;
    c->bar_seq = 0;
    // measured on 2 B200 (C3, tools/r1d.sh): the one-int NCCL allreduce barrier beat the flag
    // barrier (gather_xfer 0.17 vs 0.32 ms per epoch), so it stays the default
    const char* nb = getenv("CDFGNN_DEV_BARRIER");
    c->bar_dev = nb && atoi(nb) != 0;
    // every rank must have mapped its peers before anyone pushes
    NCCL_TRY(ncclAllReduce(c->scal_d + 4, c->scal_d + 4, 1, ncclInt32, ncclSum, c->comm, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return CDFGNN_OK;
}

void sync_args(cdfgnn_ctx* c, int l, int dir, float* const* X, int64_t ld, float eps, bool skip_gather,
               std::vector<SyncArgs>& args, bool skip_scatter = false) {
    const int F = (int)sync_width(c, l);
    const int bits = c->cfg.quant_bits;
    args.assign(c->k, SyncArgs{});
    for (int t = 0; t < c->k; ++t) {
        LocalPart& P = c->parts[t];
        SyncArgs& a = args[t];
        a.X = X[t]; a.ld = ld; a.F = F; a.eps = eps;
        a.nocache = c->cfg.cache_on ? 0 : 1;
        a.c = P.cache[l - 1][dir];
        a.stats = c->stats_d + ((l - 1) * 2 + dir) * 4;
        a.no_msgs = skip_gather ? 1 : 0;
        a.no_scatter = skip_scatter ? 1 : 0;
        a.rowb = code_row_bytes(bits, ld);
        a.stride = slot_stride(bits, ld);
        a.gstamp = c->stamp[l - 1][dir][0];
        a.sstamp = c->stamp[l - 1][dir][1];
        a.relu = (c->relu_z && dir == 0) ? 1 : 0;
    }
}

// the part's halo descriptor with the send / fired / active flags of sync (l, dir)
HaloDev halo_for(const cdfgnn_ctx* c, const LocalPart& P, int l, int dir) {
    HaloDev h = P.halo;
    const int64_t k = (int64_t)(l - 1) * 2 + dir;
    h.gflag = P.gflag + k * P.M;
    h.fired = P.fired + k * P.B;
    h.active = P.active + k * P.B;
    return h;
}

// slot layout: fresh stamps for the two phases of sync (l, dir) — every rank runs the same
// sequence of syncs, so the stamps agree across ranks
void new_stamps(cdfgnn_ctx* c, int l, int dir, int64_t ld) {
    c->stamp[l - 1][dir][0] = ++c->seq;
    c->stamp[l - 1][dir][1] = ++c->seq;
    c->last_stamp[0] = c->stamp[l - 1][dir][0];
    c->last_stamp[1] = c->stamp[l - 1][dir][1];
    c->last_ld[0] = c->last_ld[1] = ld;
}

// Gather phase of one synchronisation (Alg. 2 L3-L9): mirrors test, quantise, pack, and the
// transfer to the master parts.  Runs on `s` (the caller stream, or c->s2 when overlapped).
int halo_gather(cdfgnn_ctx* c, int l, int dir, float* const* X, int64_t ld, float eps,
                cudaStream_t s, int64_t* wire) {
    const int p = c->p;
    const int F = (int)sync_width(c, l);
    if (ld != ld_of(F)) CDF_FAIL(CDFGNN_EUSAGE, "ld %lld must equal roundup(F=%d, 4)", (long long)ld, F);
    std::vector<SyncArgs> args;
    sync_args(c, l, dir, X, ld, eps, false, args);
    const int64_t rowb = code_row_bytes(c->cfg.quant_bits, ld);
    if (c->slot) {
        // senders store straight into the masters' slots (own region co-resident, peer GPU push)
        for (int t = 0; t < c->k; ++t) {
            LocalPart& P = c->parts[t];
            c->launches += launch_gather_slot(halo_for(c, P, l, dir), args[t], P.gdst, s);
        }
        CDF_TRY(check_launch("gather_slot"));
        if (!(c->s2 && s == c->s2)) mark(c, PH_SYNC, s, SS_GXFER);
        if (c->transport == 2) CDF_TRY(push_barrier(c, s));
        return CDFGNN_OK;
    }
    for (int t = 0; t < c->k; ++t) {
        LocalPart& P = c->parts[t];
        const int nt = gather_tiles_host(P.moff.data(), p, ld);
        CUDA_TRY(cudaMemsetAsync(P.cnt, 0, sizeof(int32_t) * p, s));       // range reservations
        c->launches += launch_gather_pack_n(halo_for(c, P, l, dir), args[t], nt, s);
    }
    CDF_TRY(check_launch("gather_pack"));
    if (!(c->s2 && s == c->s2)) mark(c, PH_SYNC, s, SS_GXFER);   // no marks on the side stream
    if (c->transport == 1) CDF_TRY(nccl_phase(c, c->parts[0], true, rowb, s, wire));
    if (c->transport == 2) {
        LocalPart& P = c->parts[0];
        c->launches += launch_put(P.putG_d, p, c->hdr_bytes, rowb,
                                  *std::max_element(P.capA.begin(), P.capA.end()), s);
        CDF_TRY(check_launch("put gather"));
        CDF_TRY(push_barrier(c, s));
    }
    return CDFGNN_OK;
}

// Master apply + scatter phase (Alg. 2 L10-L22).  skip_gather: no gather ran (§8 f2).
int halo_finish(cdfgnn_ctx* c, int l, int dir, float* const* X, int64_t ld, float eps,
                cudaStream_t s, int64_t* wire, bool skip_gather, bool skip_scatter) {
    const int p = c->p;
    std::vector<SyncArgs> args;
    sync_args(c, l, dir, X, ld, eps, skip_gather, args, skip_scatter);
    const int64_t rowb = code_row_bytes(c->cfg.quant_bits, ld);
    mark(c, PH_SYNC, s, SS_MASTER);
    if (c->slot) {
        // masters apply their slots in ascending source order, their own Δ, and store the
        // scatter messages straight into the mirrors' slots (one kernel, L10-L22)
        for (int t = 0; t < c->k; ++t) {
            LocalPart& P = c->parts[t];
            c->launches += launch_master_slot(halo_for(c, P, l, dir), args[t], P.gsrc, P.sdst, s);
        }
        CDF_TRY(check_launch("master_slot"));
        if (skip_scatter) return CDFGNN_OK;
        mark(c, PH_SYNC, s, SS_SXFER);
        if (c->transport == 2) CDF_TRY(push_barrier(c, s));
        mark(c, PH_SYNC, s, SS_MIRROR);
        for (int t = 0; t < c->k; ++t) {
            LocalPart& P = c->parts[t];
            c->launches += launch_mirror_slot(halo_for(c, P, l, dir), args[t], P.ssrc, s);
        }
        return check_launch("mirror_slot");
    }
    // ---- masters: apply in ascending source order, own test, stage scatter (L10-L19)
    for (int t = 0; t < c->k; ++t) {
        LocalPart& P = c->parts[t];
        if (P.B == 0) continue;
        if (!skip_gather) {
            CUDA_TRY(cudaMemsetAsync(P.idxmap, 0xFF, sizeof(int32_t) * p * P.B, s));
            c->launches += launch_map(P.halo, P.grecv_h, 0, *std::max_element(P.capB.begin(), P.capB.end()), s);
        }
        c->launches += launch_master(halo_for(c, P, l, dir), args[t], P.grecv_h, s);
    }
    CDF_TRY(check_launch("master"));
    if (skip_scatter) return CDFGNN_OK;
    mark(c, PH_SYNC, s, SS_SPACK);
    // ---- scatter: active masters to every mirror (L20-L22)
    for (int t = 0; t < c->k; ++t) {
        LocalPart& P = c->parts[t];
        const int nt = scatter_tiles_host(P.hoff.data(), p);
        CUDA_TRY(cudaMemsetAsync(P.cnt + 2 * p, 0, sizeof(int32_t) * p, s));
        c->launches += launch_scatter_pack_n(halo_for(c, P, l, dir), args[t], nt, s);
    }
    CDF_TRY(check_launch("scatter_pack"));
    mark(c, PH_SYNC, s, SS_SXFER);
    if (c->transport == 1) CDF_TRY(nccl_phase(c, c->parts[0], false, rowb, s, wire));
    if (c->transport == 2) {
        LocalPart& P = c->parts[0];
        c->launches += launch_put(P.putS_d, p, c->hdr_bytes, rowb,
                                  *std::max_element(P.capB.begin(), P.capB.end()), s);
        CDF_TRY(check_launch("put scatter"));
        CDF_TRY(push_barrier(c, s));
    }
    mark(c, PH_SYNC, s, SS_MIRROR);
    for (int t = 0; t < c->k; ++t) {
        LocalPart& P = c->parts[t];
        if (P.M == 0) continue;
        CUDA_TRY(cudaMemsetAsync(P.mmap, 0xFF, sizeof(int32_t) * P.M, s));
        c->launches += launch_map(P.halo, P.srecv_h, 1, *std::max_element(P.capA.begin(), P.capA.end()), s);
        c->launches += launch_mirror_apply(halo_for(c, P, l, dir), args[t], P.srecv_h, s);
    }
    CDF_TRY(check_launch("mirror_apply"));
    return CDFGNN_OK;
}

// skip_gather / skip_scatter: §8 f2 dead-sync elision inside cdfgnn_epoch — the layer-L
// forward scatter (mirrors never read logits, the loss is on masters) and the
// layer-L backward gather (mirrors' δ̈^(L) is identically zero) carry no information.
int halo_impl(cdfgnn_ctx* c, int l, int dir, float* const* X, int64_t ld, float eps,
              cudaStream_t s, int64_t* wire, bool skip_gather = false, bool skip_scatter = false) {
    const int F = (int)sync_width(c, l);
    if (ld != ld_of(F)) CDF_FAIL(CDFGNN_EUSAGE, "ld %lld must equal roundup(F=%d, 4)", (long long)ld, F);
    new_stamps(c, l, dir, ld);
    mark(c, PH_SYNC, s, SS_GPACK);
    if (!skip_gather) CDF_TRY(halo_gather(c, l, dir, X, ld, eps, s, wire));
    else mark(c, PH_SYNC, s, SS_GXFER);
    return halo_finish(c, l, dir, X, ld, eps, s, wire, skip_gather, skip_scatter);
}

// The overlapped schedule applies when there is something to exchange and the transfer has no
// host round trip (NVLink push, or co-resident parts); the NCCL transport reads counts on the host.
bool overlap_on(const cdfgnn_ctx* c) { return c->cfg.overlap && c->p > 1 && c->transport != 1 && c->s2; }

// Hand the gather of (l, dir) to s2 once the caller stream has produced every mirror row.
int launch_gather_async(cdfgnn_ctx* c, int l, int dir, float* const* X, int64_t ld, float eps,
                        cudaStream_t s, int64_t* wire) {
    static const bool serial = getenv("CDFGNN_OVL_SERIAL") && atoi(getenv("CDFGNN_OVL_SERIAL"));
    cudaStream_t gs = serial ? s : c->s2;
    CUDA_TRY(cudaEventRecord(c->evA, s));
    CUDA_TRY(cudaStreamWaitEvent(gs, c->evA, 0));
    new_stamps(c, l, dir, ld);
    CDF_TRY(halo_gather(c, l, dir, X, ld, eps, gs, wire));
    CUDA_TRY(cudaEventRecord(c->evB, gs));
    c->pend[l - 1][dir] = true;
    return CDFGNN_OK;
}

// Join a gather launched by launch_gather_async, then finish the synchronisation on s.
int halo_join_finish(cdfgnn_ctx* c, int l, int dir, float* const* X, int64_t ld, float eps,
                     cudaStream_t s, int64_t* wire, bool skip_scatter) {
    mark(c, PH_SYNC, s, SS_GXFER);          // exposed (not hidden) part of the gather phase
    CUDA_TRY(cudaStreamWaitEvent(s, c->evB, 0));
    c->pend[l - 1][dir] = false;
    return halo_finish(c, l, dir, X, ld, eps, s, wire, false, skip_scatter);
}

void fill_sync_stats(const cdfgnn_ctx* c, int l, int dir, const unsigned long long* h, int64_t wire,
                     cdfgnn_sync_stats* st) {
    const int64_t F = sync_width(c, l);
    st->gather_sent = h[0];
    st->master_fired = h[1];
    st->active = h[2];
    st->scatter_msgs = h[3];
    int64_t M = 0;
    for (const LocalPart& P : c->parts) M += P.M;
    st->baseline = 2 * M;
    // O9 / R25: B·F bits of codes + 2·32 bits (lo, hi) + a 32-bit position per quantised
    // message (F + 12 bytes at B = 8), 4F + 4 bytes per fp32 message
    const int B = c->cfg.quant_bits;
    const int64_t mb = B ? (B * F + 7) / 8 + 12 : 4 * F + 4;
    st->bytes_alg = (h[0] + h[3]) * mb;
    st->bytes_wire = wire;
    if (c->transport == 2)      // NVLink push: every message is stored into a peer GPU
        st->bytes_wire = (int64_t)(h[0] + h[3]) *
                         (c->slot ? 16 + code_row_bytes(B, ld_of(F)) : c->hdr_bytes + code_row_bytes(B, ld_of(F)));
    (void)dir;
}

int read_stats_now(cdfgnn_ctx* c, int l, int dir, int64_t wire, cudaStream_t s,
                   cdfgnn_sync_stats* st) {
    unsigned long long* slot = c->stats_d + ((l - 1) * 2 + dir) * 4;
    CUDA_TRY(cudaMemcpyAsync(c->stats_h, slot, sizeof(long long) * 4, cudaMemcpyDeviceToHost, s));
    CDF_TRY(wait_stream(c, s));
    fill_sync_stats(c, l, dir, c->stats_h, wire, st);
    return CDFGNN_OK;
}

// rows: 0 = all rows (longest first), 1 = mirror rows only, 2 = master + interior rows only
int spmm_part(cdfgnn_ctx* c, LocalPart& P, const float* T, float* Y, int64_t ld, cudaStream_t s,
              int rows = 0, const GatherFuse* gf = nullptr, int64_t relu_row0 = INT64_MAX) {
    const SpmmPlan& S = spmm_plan(P, ld);
    const int64_t n = rows == 0 ? S.n_items : (rows == 1 ? S.n_items_mir : S.n_items - S.n_items_mir);
    if (n <= 0) return CDFGNN_OK;
    mark(c, PH_SPMM, s, ld);
    // column slices (CDFGNN_SPMM_CSLICE = slice width): each pass gathers an L2-sized slice of T
    const int cslice = env_knob("CDFGNN_SPMM_CSLICE", 0);
    if (cslice > 0 && ld > cslice && rows == 0 && cslice % 4 == 0 && !gf && relu_row0 == INT64_MAX) {
        for (int64_t c0 = 0; c0 < ld; c0 += cslice) {
            const int64_t w = std::min<int64_t>(ld - c0, cslice);
            const SpmmPlan& Sw = spmm_plan(P, w);
            if (Sw.nslots && w > Sw.pstride) CDF_FAIL(CDFGNN_EUSAGE, "column slice wider than the split-row scratch");
            launch_spmm(P.rowptr, P.colidx, P.val, Sw.n_items, spmm_items(P, 0, w), T + c0, Y + c0, ld, s, w);
            c->launches++;
        }
        return check_launch("spmm");
    }
    launch_spmm(P.rowptr, P.colidx, P.val, n, spmm_items(P, rows, ld), T, Y, ld, s, 0, gf, relu_row0);
    c->launches++;
    return check_launch("spmm");
}

// §8 f1: the forward SpMM runs the gather of its synchronisation in its epilogue (slot layout,
// no boundary-rows-first split; cfg.fuse_gather = 0 disables it)
bool fuse_gather_on(const cdfgnn_ctx* c) {
    return c->cfg.fuse_gather != 0 && c->slot && c->p > 1;
}

// cfg.static_inputs == 2 (hoisted input aggregation): X is fixed per buffer, so the
// layer-1 product Â_i X_i W^(0) of eq. (1) is evaluated as (Â_i X_i) W^(0) with Â_i X_i
// aggregated once per X pointer (associativity), and ∇W^(0) = X_iᵀ (Â_i δ^(1))
// (reading R6) as (Â_i X_i)ᵀ δ^(1) (Â_i symmetric) — both layer-1 SpMMs leave
// the epoch.  Results agree with the per-epoch schedule up to fp32 rounding order.
bool hoisted(const cdfgnn_ctx* c, int l) { return l == 1 && c->cfg.static_inputs == 2; }

// ∇W from MN-major H and S in place (default) or from transposed K-major copies
// (CDFGNN_WGRAD_KMAJOR=1, the earlier path)
bool wgrad_mn() {
    static const bool v = [] { const char* e = getenv("CDFGNN_WGRAD_KMAJOR"); return !(e && atoi(e) != 0); }();
    return v;
}

int ensure_ax(cdfgnn_ctx* c, LocalPart& P, const float* X, int64_t ld_in, cudaStream_t s) {
    if (P.ax_src == X) return CDFGNN_OK;
    const int64_t F0 = c->cfg.dims[0];
    if (ld_in != ld_of(F0)) CDF_FAIL(CDFGNN_EUSAGE, "hoisted input aggregation needs ld(X) = %lld",
                                     (long long)ld_of(F0));
    // the SpMM kernels cover <= 1024 columns per launch: wider inputs (C1's 1433 features)
    // are aggregated in 1024-column slices of the same rows
    const int64_t w0 = std::min<int64_t>(ld_in, 1024);
    const SpmmPlan& S = spmm_plan(P, w0);
    if (S.nslots && w0 > S.pstride) CDF_FAIL(CDFGNN_EUSAGE, "split SpMM rows cannot hold width %lld",
                                             (long long)w0);
    mark(c, PH_OTHER, s);
    for (int64_t c0 = 0; c0 < ld_in; c0 += 1024) {
        const int64_t w = std::min<int64_t>(ld_in - c0, 1024);
        launch_spmm(P.rowptr, P.colidx, P.val, S.n_items, spmm_items(P, 0, w0), X + c0, P.ax + c0, ld_in, s, w);
        c->launches++;
    }
    CDF_TRY(check_launch("spmm (input aggregation)"));
    if (P.xT && !wgrad_mn()) {
        c->launches += launch_transpose(P.ax, P.n, F0, ld_in, P.xT, ld_of(P.n), s);
        P.xT_src = P.ax;
    }
    P.ax_src = X;
    return CDFGNN_OK;
}

int fwd_impl(cdfgnn_ctx* c, int l, const float* const* H_in, int64_t ld_in, const float* W,
             float* const* Z, float* const* H_out, int64_t ld_out, float eps, cudaStream_t s,
             int64_t* wire, bool elide = false) {
    const int64_t Fi = c->cfg.dims[l - 1], Fo = c->cfg.dims[l];
    if (ld_in < Fi || ld_in % 4 || ld_out != ld_of(Fo)) CDF_FAIL(CDFGNN_EUSAGE, "bad leading dimension");
    float* Wt = c->wtpad + c->wtoff[l - 1];
    const int64_t ldwt = ld_of(Fi);
    const bool hz = hoisted(c, l);
    const bool ov = overlap_on(c) && !hz;
    if (c->cfg.gemm_tf32) {
        mark(c, PH_GEMM, s);
        c->launches += launch_transpose(W, Fi, Fo, Fo, Wt, ldwt, s);
    }
    const bool fuse = !ov && !hz && fuse_gather_on(c) && env_knob("CDFGNN_SPMM_CSLICE", 0) == 0;
    // σ fused (R3): in place (H_out == Z), interior rows by the SpMM epilogue, boundary rows by the
    // slot-layout master / mirror kernels; the K-major Hᵀ path and the hoisted layer keep the
    // separate ReLU
    bool frelu = H_out && !hz && (c->slot || c->p == 1) && env_knob("CDFGNN_SPMM_CSLICE", 0) == 0 &&
                 env_knob("CDFGNN_FUSE_RELU", 1) != 0;
    for (int t = 0; frelu && t < c->k; ++t)
        frelu = H_out[t] == Z[t] && !(c->parts[t].hT[l] && c->in_epoch && !wgrad_mn());
    std::vector<SyncArgs> fargs;
    if (fuse) {
        if (ld_out != ld_of(Fo)) CDF_FAIL(CDFGNN_EUSAGE, "ld %lld must equal roundup(F, 4)", (long long)ld_out);
        new_stamps(c, l, 0, ld_out);
        sync_args(c, l, 0, Z, ld_out, eps, false, fargs);
    }
    for (int t = 0; t < c->k; ++t) {
        LocalPart& P = c->parts[t];
        const float* A = H_in[t];
        if (hz) {
            CDF_TRY(ensure_ax(c, P, H_in[t], ld_in, s));
            A = P.ax;
        }
        float* out = hz ? Z[t] : P.T;      // hoisted: the GEMM yields Z̈ directly
        mark(c, PH_GEMM, s);
        if (c->cfg.gemm_tf32) {
            CDF_TRY(gemm_tc_fwd(P.n, Fo, Fi, A, ld_in, Wt, ldwt, out, ld_out, c->cfg.gemm_tf32 == 3, s));
        } else {
            launch_gemm_simt(false, false, P.n, Fo, Fi, A, ld_in, W, Fo, out, ld_out, nullptr, 0,
                             nullptr, 0, false, s);
        }
        c->launches++;
        CDF_TRY(check_launch("gemm fwd"));
        const int64_t r0 = frelu ? P.B + P.M : INT64_MAX;
        if (fuse) {
            GatherFuse gf;
            gf.h = halo_for(c, P, l, 0);
            gf.a = fargs[t];
            gf.dst = P.gdst;
            CDF_TRY(spmm_part(c, P, P.T, Z[t], ld_out, s, 0, &gf, r0));
        } else if (!hz) {
            CDF_TRY(spmm_part(c, P, P.T, Z[t], ld_out, s, ov ? 1 : 0, nullptr, r0));
        }
    }
    c->relu_z = frelu;
    if (fuse) {
        // the gather ran in the SpMM epilogues: count its senders, transfer barrier, then the
        // master apply and scatter (Alg. 2 L10-L22)
        mark(c, PH_SYNC, s, SS_GPACK);
        for (int t = 0; t < c->k; ++t) {
            LocalPart& P = c->parts[t];
            launch_count_flags(halo_for(c, P, l, 0).gflag, P.M, fargs[t].stats, s);
            c->launches++;
        }
        CDF_TRY(check_launch("count_flags"));
        mark(c, PH_SYNC, s, SS_GXFER);
        if (c->transport == 2) CDF_TRY(push_barrier(c, s));
        CDF_TRY(halo_finish(c, l, 0, Z, ld_out, eps, s, wire, false, elide && l == c->cfg.L));
    } else if (ov) {
        // §8 f1: the mirror rows are done — their gather runs on s2 under the remaining SpMM rows
        CDF_TRY(launch_gather_async(c, l, 0, Z, ld_out, eps, s, wire));
        for (int t = 0; t < c->k; ++t)
            CDF_TRY(spmm_part(c, c->parts[t], c->parts[t].T, Z[t], ld_out, s, 2, nullptr,
                              frelu ? c->parts[t].B + c->parts[t].M : INT64_MAX));
        CDF_TRY(halo_join_finish(c, l, 0, Z, ld_out, eps, s, wire, elide && l == c->cfg.L));
    } else {
        CDF_TRY(halo_impl(c, l, 0, Z, ld_out, eps, s, wire, false, elide && l == c->cfg.L));
    }
    c->relu_z = false;
    if (H_out && !frelu) {
        mark(c, PH_OTHER, s);
        for (int t = 0; t < c->k; ++t) {
            LocalPart& P = c->parts[t];
            if (P.hT[l] && c->in_epoch && !wgrad_mn()) {
                // ReLU fused with the transpose the next layer's ∇W needs (K-major Hᵀ)
                c->launches += launch_relu_transpose(Z[t], P.n, Fo, ld_out, H_out[t], P.hT[l], ld_of(P.n), s);
                P.hT_src[l] = H_out[t];
            } else {
                launch_relu(Z[t], H_out[t], P.n * ld_out, s);
                c->launches++;
            }
        }
        CDF_TRY(check_launch("relu"));
    }
    return CDFGNN_OK;
}

// wire_prev: transfer counter of the (l-1, δ) sync, whose gather this call may launch early
int bwd_impl(cdfgnn_ctx* c, int l, float* const* dZ, int64_t ld, const float* const* H_in,
             int64_t ld_in, const float* W, float* const* dZ_prev, float* dW, float eps,
             cudaStream_t s, int64_t* wire, bool elide = false, int64_t* wire_prev = nullptr) {
    const int64_t Fi = c->cfg.dims[l - 1], Fo = c->cfg.dims[l];
    if (ld != ld_of(Fo) || ld_in < Fi || ld_in % 4) CDF_FAIL(CDFGNN_EUSAGE, "bad leading dimension");
    if (c->pend[l - 1][1]) CDF_TRY(halo_join_finish(c, l, 1, dZ, ld, eps, s, wire, false));
    else CDF_TRY(halo_impl(c, l, 1, dZ, ld, eps, s, wire, elide && l == c->cfg.L, false));
    // §8 f1 in the backward pass: δ̈^(l-1) mirror rows first, their gather on s2 under ∇W and
    // the remaining rows (inside cdfgnn_epoch, where the next call joins it)
    const bool ov = dZ_prev && c->in_epoch && overlap_on(c) && ld_in == ld_of(Fi);
    // δ̈^(l-1) rows [r0, r1) of part t: (S Wᵀ) ⊙ 𝟙[H > 0]
    auto bwd_data_rows = [&](int t, int64_t r0, int64_t r1) -> int {
        LocalPart& P = c->parts[t];
        if (r1 <= r0) return CDFGNN_OK;
        if (c->cfg.gemm_tf32) {
            CDF_TRY(gemm_tc_bwd_data(r1 - r0, Fi, Fo, P.S + r0 * ld, ld, c->wpad + c->wpoff[l - 1], ld,
                                     dZ_prev[t] + r0 * ld_in, ld_in, H_in[t] + r0 * ld_in, ld_in,
                                     c->cfg.gemm_tf32 == 3, s));
        } else {
            launch_gemm_simt(false, true, r1 - r0, Fi, Fo, P.S + r0 * ld, ld, W, Fo, dZ_prev[t] + r0 * ld_in,
                             ld_in, H_in[t] + r0 * ld_in, ld_in, nullptr, 0, false, s);
        }
        c->launches++;
        return check_launch("gemm bwd_data");
    };
    const bool hz = hoisted(c, l);
    for (int t = 0; t < c->k; ++t) {
        LocalPart& P = c->parts[t];
        if (hz) {
            CDF_TRY(ensure_ax(c, P, H_in[t], ld_in, s));   // no SpMM: ∇W^(0) = (Â_i X_i)ᵀ δ^(1)
            continue;
        }
        CDF_TRY(spmm_part(c, P, dZ[t], P.S, ld, s));
        mark(c, PH_GEMM, s);
        if (c->cfg.gemm_tf32 && t == 0)
            c->launches += launch_pad_rows(W, Fi, Fo, c->wpad + c->wpoff[l - 1], ld, s);
        if (ov) CDF_TRY(bwd_data_rows(t, P.B, P.B + P.M));
    }
    if (ov) CDF_TRY(launch_gather_async(c, l - 1, 1, dZ_prev, ld_in, eps, s, wire_prev));
    for (int t = 0; t < c->k; ++t) {
        LocalPart& P = c->parts[t];
        mark(c, PH_GEMM, s);
        // dW (+)= H_inᵀ S ; parts accumulate in ascending order
        const float* Sg = hz ? dZ[t] : P.S;      // hoisted layer 1: (Â_i X_i)ᵀ δ^(1)
        const float* Hg = hz ? P.ax : H_in[t];
        if (c->cfg.gemm_tf32 && wgrad_mn()) {
            CDF_TRY(gemm_tc_wgrad_mn(Fi, Fo, P.n, Hg, ld_in, Sg, ld, dW, Fo, c->splitk, c->splitk_cap, t > 0,
                                     c->cfg.gemm_tf32 == 3, s, &c->launches));
        } else if (c->cfg.gemm_tf32) {
            const float* Ht = c->trA;
            int64_t ldh = c->npad;
            if (hz && P.xT) {
                Ht = P.xT;                      // (Â_i X_i)ᵀ, built by ensure_ax
                ldh = ld_of(P.n);
            } else if (hz) {
                c->launches += launch_transpose(P.ax, P.n, Fi, ld_in, c->trA, c->npad, s);
            } else if (l == 1 && P.xT) {
                // static inputs: H^(0)ᵀ = Xᵀ is transposed once per X buffer and reused
                if (P.xT_src != H_in[t]) {
                    c->launches += launch_transpose(H_in[t], P.n, Fi, ld_in, P.xT, ld_of(P.n), s);
                    P.xT_src = H_in[t];
                }
                Ht = P.xT;
                ldh = ld_of(P.n);
            } else if (l >= 2 && c->in_epoch && P.hT[l - 1] && P.hT_src[l - 1] == H_in[t]) {
                Ht = P.hT[l - 1];               // written by the forward ReLU of layer l-1
                ldh = ld_of(P.n);
            } else {
                c->launches += launch_transpose(H_in[t], P.n, Fi, ld_in, c->trA, c->npad, s);
            }
            c->launches += launch_transpose(Sg, P.n, Fo, ld, c->trB, c->npad, s);
            CDF_TRY(gemm_tc_wgrad(Fi, Fo, P.n, Ht, ldh, c->trB, c->npad, dW, Fo, c->splitk,
                                  c->splitk_cap, t > 0, c->cfg.gemm_tf32 == 3, s, &c->launches));
        } else {
            launch_gemm_simt(true, false, Fi, Fo, P.n, Hg, ld_in, Sg, ld, dW, Fo, nullptr, 0,
                             c->splitk, c->splitk_cap, t > 0, s);
            c->launches += 2;
        }
        CDF_TRY(check_launch("gemm wgrad"));
        if (t == c->k - 1 && c->in_epoch && c->comm_grad) {
            // ∇W^(l-1) is final on this rank: sum it over the ranks on the side stream while the
            // remaining backward (δ̈^(l-1), the layer l-1 sync, SpMM and GEMMs) runs on s
            CUDA_TRY(cudaEventRecord(c->evG, s));
            CUDA_TRY(cudaStreamWaitEvent(c->s3, c->evG, 0));
            NCCL_TRY(ncclAllReduce(dW, dW, (size_t)(Fi * Fo), ncclFloat32, ncclSum, c->comm_grad, c->s3));
            c->dw_pending = true;
        }
        if (dZ_prev) {
            if (ov) {
                CDF_TRY(bwd_data_rows(t, 0, P.B));
                CDF_TRY(bwd_data_rows(t, P.B + P.M, P.n));
            } else {
                CDF_TRY(bwd_data_rows(t, 0, P.n));
            }
        }
    }
    return CDFGNN_OK;
}

double update_eps(const cdfgnn_cfg& g, double eps, double acc, double mean) {
    // P:L387-393, literal, then the R17 clamp
    if (acc < mean - g.mu1 && eps < g.nu1) eps = std::min(g.lam1 * eps, eps + g.xi);
    else if (acc > mean + g.mu2 && eps > g.nu2) eps = std::max(g.lam2 * eps, eps - g.xi);
    if (g.eps_clamp) eps = std::min(std::max(eps, g.nu2), g.nu1);
    return eps;
}

}  // namespace

// =====================================================================================
extern "C" int cdfgnn_cfg_default(cdfgnn_cfg* cfg) {
    if (!cfg) CDF_FAIL(CDFGNN_EUSAGE, "cfg is NULL");
    std::memset(cfg, 0, sizeof(*cfg));
    cfg->L = 2;
    cfg->dims[0] = 16; cfg->dims[1] = 16; cfg->dims[2] = 7;
    cfg->cache_on = 1;
    cfg->eps_init = 0.01;
    cfg->adaptive = 1;
    cfg->mu1 = 0.001; cfg->mu2 = 0.02; cfg->nu1 = 0.3; cfg->nu2 = 0.001;
    cfg->xi = 0.01; cfg->lam1 = 1.05; cfg->lam2 = 0.9;
    cfg->eps_clamp = 1;
    cfg->quant_bits = 8;
    cfg->optimizer = 1;
    cfg->lr = 0.01; cfg->beta1 = 0.9; cfg->beta2 = 0.999; cfg->adam_eps = 1e-8;
    cfg->gemm_tf32 = 3;
    cfg->timing = 0;
    cfg->transport = 0;
    cfg->elide_dead_syncs = 1;
    cfg->static_inputs = 0;
    cfg->overlap = 0;
    cfg->msg_layout = 0;
    cfg->fuse_gather = 1;
    return CDFGNN_OK;
}

extern "C" int cdfgnn_get_unique_id(void* out128) {
    if (!out128) CDF_FAIL(CDFGNN_EUSAGE, "out is NULL");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId must be 128 bytes");
    ncclUniqueId id;
    NCCL_TRY(ncclGetUniqueId(&id));
    std::memcpy(out128, &id, sizeof(id));
    return CDFGNN_OK;
}

extern "C" int cdfgnn_workspace_size(const cdfgnn_plan* plan, const int32_t* parts, int32_t k,
                                     const cdfgnn_cfg* cfg, size_t* bytes) {
    if (!bytes || !parts) CDF_FAIL(CDFGNN_EUSAGE, "NULL argument");
    cdfgnn_ctx c;
    CDF_TRY(prepare(&c, plan, parts, k, cfg));
    Bump b;
    carve(&c, b);
    *bytes = align_up((int64_t)b.off, 256);
    return CDFGNN_OK;
}

extern "C" int cdfgnn_init(const cdfgnn_plan* plan, const int32_t* parts, int32_t k, int32_t rank,
                           int32_t world, const void* nccl_uid, int32_t device, void* workspace,
                           size_t workspace_bytes, const cdfgnn_cfg* cfg, cdfgnn_ctx** out) {
    if (!out || !parts || !workspace) CDF_FAIL(CDFGNN_EUSAGE, "NULL argument");
    *out = nullptr;
    if (((uintptr_t)workspace) % 256) CDF_FAIL(CDFGNN_EUSAGE, "workspace must be 256-byte aligned");
    std::unique_ptr<cdfgnn_ctx> c(new cdfgnn_ctx());
    CDF_TRY(prepare(c.get(), plan, parts, k, cfg));
    if (world < 1 || rank < 0 || rank >= world) CDF_FAIL(CDFGNN_EUSAGE, "bad rank/world");
    if (world == 1) {
        if (k != c->p) CDF_FAIL(CDFGNN_EUSAGE, "world == 1 requires all %d parts local (k = %d)", c->p, k);
        for (int t = 0; t < k; ++t)
            if (parts[t] != t) CDF_FAIL(CDFGNN_EUSAGE, "parts must be 0..p-1 in order");
    } else {
        if (k != 1 || world != c->p || parts[0] != rank)
            CDF_FAIL(CDFGNN_EUSAGE, "world > 1 requires one partition per rank (part == rank, p == world)");
        if (!nccl_uid) CDF_FAIL(CDFGNN_EUSAGE, "nccl_uid required for world > 1");
    }
    c->rank = rank; c->world = world; c->device = device;
    Bump b;
    carve(c.get(), b);
    const size_t need = align_up((int64_t)b.off, 256);
    if (workspace_bytes < need)
        CDF_FAIL(CDFGNN_EWORKSPACE, "workspace too small: %zu < %zu", workspace_bytes, need);
    c->ws = workspace; c->ws_bytes = workspace_bytes;
    b = Bump{};
    b.base = reinterpret_cast<uint8_t*>(workspace);
    carve(c.get(), b);
    CUDA_TRY(cudaSetDevice(device));
    build_tables(c.get());
    cudaStream_t s = nullptr;
    CUDA_TRY(cudaMemsetAsync(workspace, 0, need, s));
    for (LocalPart& P : c->parts) {
        CUDA_TRY(cudaMemcpyAsync(P.rowptr, P.rowptr_h, sizeof(int32_t) * (P.n + 1), cudaMemcpyHostToDevice, s));
        CUDA_TRY(cudaMemcpyAsync(P.colidx, P.colidx_h, sizeof(int32_t) * P.nnz, cudaMemcpyHostToDevice, s));
        CUDA_TRY(cudaMemcpyAsync(P.val, P.val_h, sizeof(float) * P.nnz, cudaMemcpyHostToDevice, s));
        for (SpmmPlan& S : P.sp) {
            CUDA_TRY(cudaMemcpyAsync(S.items, S.items_h.data(), sizeof(int2) * S.n_items, cudaMemcpyHostToDevice, s));
            CUDA_TRY(cudaMemcpyAsync(S.items2, S.items2_h.data(), sizeof(int2) * S.n_items, cudaMemcpyHostToDevice, s));
            CUDA_TRY(cudaMemcpyAsync(S.split, S.split_h.data(), sizeof(int4) * P.n, cudaMemcpyHostToDevice, s));
            CUDA_TRY(cudaMemcpyAsync(S.seg_beg, S.seg_beg_h.data(), sizeof(int32_t) * S.seg_beg_h.size(),
                                     cudaMemcpyHostToDevice, s));
        }
        CUDA_TRY(cudaStreamSynchronize(s));
        CUDA_TRY(cudaMemcpyAsync(P.halo_local, P.halo_h, sizeof(int32_t) * P.hoff[c->p], cudaMemcpyHostToDevice, s));
        CUDA_TRY(cudaMemcpyAsync(P.moff_d, P.moff.data(), sizeof(int64_t) * (c->p + 1), cudaMemcpyHostToDevice, s));
        CUDA_TRY(cudaMemcpyAsync(P.hoff_d, P.hoff.data(), sizeof(int64_t) * (c->p + 1), cudaMemcpyHostToDevice, s));
        CUDA_TRY(cudaMemcpyAsync(P.gsend_d, &P.gsend_h, sizeof(RegionTab), cudaMemcpyHostToDevice, s));
        CUDA_TRY(cudaMemcpyAsync(P.grecv_d, &P.grecv_h, sizeof(RegionTab), cudaMemcpyHostToDevice, s));
        CUDA_TRY(cudaMemcpyAsync(P.ssend_d, &P.ssend_h, sizeof(RegionTab), cudaMemcpyHostToDevice, s));
        CUDA_TRY(cudaMemcpyAsync(P.srecv_d, &P.srecv_h, sizeof(RegionTab), cudaMemcpyHostToDevice, s));
        CUDA_TRY(cudaMallocHost(&P.cnt_h, sizeof(int32_t) * 4 * c->p));
    }
    CUDA_TRY(cudaMallocHost(&c->stats_h, sizeof(long long) * CDFGNN_MAX_LAYERS * 2 * 4));
    CUDA_TRY(cudaMallocHost(&c->host_scratch, sizeof(double) * (c->k + 8)));
    CUDA_TRY(cudaStreamSynchronize(s));
    c->transport = 0;
    if (world > 1) {
        ncclUniqueId id;
        std::memcpy(&id, nccl_uid, sizeof(id));
        NCCL_TRY(ncclCommInitRank(&c->comm, world, id, rank));
        NCCL_TRY(ncclCommSplit(c->comm, 0, rank, &c->comm_in, nullptr));
        const char* dwo = getenv("CDFGNN_DW_OVERLAP");      // 0: one grouped allreduce after the backward
        if (!(dwo && atoi(dwo) == 0)) {
            NCCL_TRY(ncclCommSplit(c->comm, 0, rank, &c->comm_grad, nullptr));
            int plo = 0, phi = 0;
            CUDA_TRY(cudaDeviceGetStreamPriorityRange(&plo, &phi));
            CUDA_TRY(cudaStreamCreateWithPriority(&c->s3, cudaStreamNonBlocking, phi));
            CUDA_TRY(cudaEventCreateWithFlags(&c->evG, cudaEventDisableTiming));
            CUDA_TRY(cudaEventCreateWithFlags(&c->evJ, cudaEventDisableTiming));
        }
        {
            // establish the input-distribution peer connections now (NCCL connects p2p lazily,
            // which would otherwise land inside the first pipelined epochs)
            float* tmp = reinterpret_cast<float*>(c->splitk);
            NCCL_TRY(ncclGroupStart());
            for (int q = 0; q < world; ++q) {
                if (q == rank) continue;
                NCCL_TRY(ncclSend(tmp, 1, ncclFloat32, q, c->comm_in, s));
                NCCL_TRY(ncclRecv(tmp + 1 + q, 1, ncclFloat32, q, c->comm_in, s));
            }
            NCCL_TRY(ncclGroupEnd());
            CUDA_TRY(cudaStreamSynchronize(s));
        }
        c->transport = 1;
        if (cfg->transport == 0) {
            // all ranks must agree: push only if every rank mapped its peers
            int ok = setup_push(c.get(), s) == CDFGNN_OK ? 1 : 0;
            int32_t* flag = c->scal_d + 5;
            CUDA_TRY(cudaMemcpyAsync(flag, &ok, sizeof(int), cudaMemcpyHostToDevice, s));
            NCCL_TRY(ncclAllReduce(flag, flag, 1, ncclInt32, ncclMin, c->comm, s));
            CUDA_TRY(cudaMemcpyAsync(&ok, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
            CUDA_TRY(cudaStreamSynchronize(s));
            if (ok) {
                c->transport = 2;
            } else {
                // restore the NCCL send tables
                build_tables(c.get());
                LocalPart& P = c->parts[0];
                CUDA_TRY(cudaMemcpy(P.gsend_d, &P.gsend_h, sizeof(RegionTab), cudaMemcpyHostToDevice));
                CUDA_TRY(cudaMemcpy(P.ssend_d, &P.ssend_h, sizeof(RegionTab), cudaMemcpyHostToDevice));
                for (void* m : c->peer_maps) cudaIpcCloseMemHandle(m);
                c->peer_maps.clear();
                c->bar_dev = false;
            }
        }
    }
    // message layout: slot-addressed for co-resident parts and the NVLink push transport
    // (msg_layout 0 = auto, 2 = slot), compacted for NCCL send/recv (and msg_layout 1)
    if (cfg->msg_layout == 2 && c->transport == 1)
        CDF_FAIL(CDFGNN_EUSAGE, "msg_layout = 2 (slot) needs co-resident parts or the NVLink push transport");
    c->slot = cfg->msg_layout == 2 || (cfg->msg_layout == 0 && c->transport != 1);
    for (LocalPart& P : c->parts) {
        if (P.B > 0)
            CUDA_TRY(cudaMemcpyAsync(P.hpos, P.hpos_h.data(), sizeof(int32_t) * P.hpos_h.size(),
                                     cudaMemcpyHostToDevice, s));
        P.halo.remote = (c->slot && c->transport == 2) ? 1 : 0;   // kernels store into peer GPUs
    }
    CUDA_TRY(cudaStreamSynchronize(s));
    if (cfg->overlap && c->p > 1) {
        int lo = 0, hi = 0;
        CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        CUDA_TRY(cudaStreamCreateWithPriority(&c->s2, cudaStreamNonBlocking, hi));
        CUDA_TRY(cudaEventCreateWithFlags(&c->evA, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&c->evB, cudaEventDisableTiming));
    }
    c->eps = cfg->eps_init;
    c->timing = cfg->timing != 0;
    *out = c.release();
    return CDFGNN_OK;
}

extern "C" int cdfgnn_destroy(cdfgnn_ctx* c) {
    if (!c) return CDFGNN_OK;
    if (!c->peer_maps.empty()) cudaDeviceSynchronize();
    for (void* m : c->peer_maps) cudaIpcCloseMemHandle(m);
    if (c->comm_in) ncclCommDestroy(c->comm_in);
    if (c->s3) {
        cudaStreamSynchronize(c->s3);
        cudaStreamDestroy(c->s3);
    }
    if (c->evG) cudaEventDestroy(c->evG);
    if (c->evJ) cudaEventDestroy(c->evJ);
    if (c->comm_grad) ncclCommDestroy(c->comm_grad);
    if (c->comm) ncclCommDestroy(c->comm);
    for (LocalPart& P : c->parts)
        if (P.cnt_h) cudaFreeHost(P.cnt_h);
    if (c->stats_h) cudaFreeHost(c->stats_h);
    if (c->host_scratch) cudaFreeHost(c->host_scratch);
    for (cudaEvent_t e : c->ev) cudaEventDestroy(e);
    if (c->s2) {
        cudaStreamSynchronize(c->s2);
        cudaStreamDestroy(c->s2);
    }
    if (c->evA) cudaEventDestroy(c->evA);
    if (c->evB) cudaEventDestroy(c->evB);
    if (c->cs) {
        cudaStreamSynchronize(c->cs);
        cudaStreamDestroy(c->cs);
    }
    for (int i = 0; i < 2; ++i) {
        if (c->staged[i]) cudaEventDestroy(c->staged[i]);
        if (c->used[i]) cudaEventDestroy(c->used[i]);
    }
    delete c;
    return CDFGNN_OK;
}

extern "C" int cdfgnn_halo_exchange(cdfgnn_ctx* c, int32_t l, int32_t dir, float* const* X,
                                    int64_t ld, float eps, cdfgnn_sync_stats* st, void* stream) {
    if (!c || !X) CDF_FAIL(CDFGNN_EUSAGE, "NULL argument");
    if (l < 1 || l > c->cfg.L || dir < 0 || dir > 1) CDF_FAIL(CDFGNN_EUSAGE, "bad layer/dir");
    cudaStream_t s = (cudaStream_t)stream;
    c->relu_z = false;
    CUDA_TRY(cudaSetDevice(c->device));
    unsigned long long* slot = c->stats_d + ((l - 1) * 2 + dir) * 4;
    if (st) CUDA_TRY(cudaMemsetAsync(slot, 0, sizeof(long long) * 4, s));
    int64_t wire = 0;
    CDF_TRY(halo_impl(c, l, dir, X, ld, eps, s, &wire));
    if (st) CDF_TRY(read_stats_now(c, l, dir, wire, s, st));
    return CDFGNN_OK;
}

extern "C" int cdfgnn_layer_fwd(cdfgnn_ctx* c, int32_t l, const float* const* H_in, int64_t ld_in,
                                const float* W, float* const* Z, float* const* H_out, int64_t ld_out,
                                float eps, cdfgnn_sync_stats* st, void* stream) {
    if (!c || !H_in || !W || !Z) CDF_FAIL(CDFGNN_EUSAGE, "NULL argument");
    if (l < 1 || l > c->cfg.L) CDF_FAIL(CDFGNN_EUSAGE, "bad layer");
    cudaStream_t s = (cudaStream_t)stream;
    c->relu_z = false;
    CUDA_TRY(cudaSetDevice(c->device));
    unsigned long long* slot = c->stats_d + ((l - 1) * 2) * 4;
    if (st) CUDA_TRY(cudaMemsetAsync(slot, 0, sizeof(long long) * 4, s));
    int64_t wire = 0;
    CDF_TRY(fwd_impl(c, l, H_in, ld_in, W, Z, H_out, ld_out, eps, s, &wire));
    if (st) CDF_TRY(read_stats_now(c, l, 0, wire, s, st));
    return CDFGNN_OK;
}

extern "C" int cdfgnn_layer_bwd(cdfgnn_ctx* c, int32_t l, float* const* dZ, int64_t ld,
                                const float* const* H_in, int64_t ld_in, const float* W,
                                float* const* dZ_prev, float* dW, float eps,
                                cdfgnn_sync_stats* st, void* stream) {
    if (!c || !dZ || !H_in || !W || !dW) CDF_FAIL(CDFGNN_EUSAGE, "NULL argument");
    if (l < 1 || l > c->cfg.L) CDF_FAIL(CDFGNN_EUSAGE, "bad layer");
    cudaStream_t s = (cudaStream_t)stream;
    c->relu_z = false;
    CUDA_TRY(cudaSetDevice(c->device));
    unsigned long long* slot = c->stats_d + ((l - 1) * 2 + 1) * 4;
    if (st) CUDA_TRY(cudaMemsetAsync(slot, 0, sizeof(long long) * 4, s));
    int64_t wire = 0;
    CDF_TRY(bwd_impl(c, l, dZ, ld, H_in, ld_in, W, dZ_prev, dW, eps, s, &wire));
    if (st) CDF_TRY(read_stats_now(c, l, 1, wire, s, st));
    return CDFGNN_OK;
}

static int epoch_impl(cdfgnn_ctx* c, const float* const* X, const int32_t* const* labels,
                      const uint8_t* const* train, float* const* W, cdfgnn_epoch_stats* out,
                      cudaStream_t s) {
    const int L = c->cfg.L, k = c->k;
    const int C = c->cfg.dims[L];
    c->relu_z = false;
    c->launches = 0;
    c->ev_used = 0;
    std::memset(c->pend, 0, sizeof(c->pend));
    if (c->dw_pending) {               // an earlier epoch failed between a ∇W allreduce and the join
        CUDA_TRY(cudaEventRecord(c->evJ, c->s3));
        CUDA_TRY(cudaStreamWaitEvent(s, c->evJ, 0));
        c->dw_pending = false;
    }
    int64_t wire[CDFGNN_MAX_LAYERS][2] = {};
    CUDA_TRY(cudaMemsetAsync(c->stats_d, 0, sizeof(long long) * CDFGNN_MAX_LAYERS * 2 * 4, s));
    CUDA_TRY(cudaMemsetAsync(c->scal_d, 0, sizeof(int32_t) * 8, s));
    mark(c, PH_OTHER, s);
    if (c->ntrain < 0) {
        // global train count over masters (every train vertex has exactly one master)
        for (int t = 0; t < k; ++t) {
            LocalPart& P = c->parts[t];
            launch_count_train(P.n, P.B, P.M, train[t], c->scal_d + 2, s);
            c->launches++;
        }
        if (c->world > 1)
            NCCL_TRY(ncclAllReduce(c->scal_d + 2, c->scal_d + 2, 1, ncclInt32, ncclSum, c->comm, s));
        int32_t* hs = reinterpret_cast<int32_t*>(c->host_scratch);
        CUDA_TRY(cudaMemcpyAsync(hs, c->scal_d + 2, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        CDF_TRY(wait_stream(c, s));
        c->ntrain = hs[0];
        if (c->ntrain <= 0) CDF_FAIL(CDFGNN_EDATA, "no training vertices");
    }
    const double eps_used = c->cfg.cache_on ? c->eps : 0.0;
    const float eps32 = (float)eps_used;   // reading R15: rounded once on the host
    // ---- forward (Alg. 1 L2-L6)
    std::vector<const float*> hin(k);
    for (int t = 0; t < k; ++t) hin[t] = X[t];
    int64_t ld_in = ld_of(c->cfg.dims[0]);
    for (int l = 1; l <= L; ++l) {
        const int64_t ld = ld_of(c->cfg.dims[l]);
        std::vector<float*> z(k);
        for (int t = 0; t < k; ++t) z[t] = c->parts[t].act[l];
        CDF_TRY(fwd_impl(c, l, hin.data(), ld_in, W[l - 1], z.data(), l < L ? z.data() : nullptr,
                         ld, eps32, s, &wire[l - 1][0], c->cfg.elide_dead_syncs != 0));
        for (int t = 0; t < k; ++t) hin[t] = z[t];
        ld_in = ld;
    }
    // ---- loss on masters (Alg. 1 L7)
    mark(c, PH_OTHER, s);
    const int64_t ldL = ld_of(C);
    std::vector<float*> dcur(k), dprev(k);
    for (int t = 0; t < k; ++t) {
        LocalPart& P = c->parts[t];
        launch_loss(P.act[L], ldL, C, P.n, P.B, P.M, labels[t], train[t], 1.0 / (double)c->ntrain,
                    P.D[L & 1], P.rowloss, c->scal_d, c->scal_d + 1, s);
        launch_reduce_rows(P.rowloss, P.n, c->loss_d + t, c->loss_part, s);
        c->launches += 3;
        dcur[t] = P.D[L & 1];
    }
    CDF_TRY(check_launch("loss"));
    // ---- backward (Alg. 1 L8-L14)
    for (int l = L; l >= 1; --l) {
        const int64_t ld = ld_of(c->cfg.dims[l]);
        const int64_t ldi = ld_of(c->cfg.dims[l - 1]);
        std::vector<const float*> h(k);
        for (int t = 0; t < k; ++t) {
            h[t] = l == 1 ? X[t] : c->parts[t].act[l - 1];
            dprev[t] = c->parts[t].D[(l - 1) & 1];
        }
        CDF_TRY(bwd_impl(c, l, dcur.data(), ld, h.data(), ldi, W[l - 1], l > 1 ? dprev.data() : nullptr,
                         c->dW + c->woff[l - 1], eps32, s, &wire[l - 1][1], c->cfg.elide_dead_syncs != 0,
                         l > 1 ? &wire[l - 2][1] : nullptr));
        dcur = dprev;
    }
    // ---- parameter aggregation + update (Alg. 1 L12-L13)
    mark(c, PH_OTHER, s);
    if (c->dw_pending) {
        CUDA_TRY(cudaEventRecord(c->evJ, c->s3));     // join the per-layer ∇W allreduces
        CUDA_TRY(cudaStreamWaitEvent(s, c->evJ, 0));
        c->dw_pending = false;
    }
    if (c->world > 1) {
        NCCL_TRY(ncclGroupStart());
        if (!c->comm_grad)
            NCCL_TRY(ncclAllReduce(c->dW, c->dW, (size_t)c->wtotal, ncclFloat32, ncclSum, c->comm, s));
        NCCL_TRY(ncclAllReduce(c->loss_d, c->loss_d, 1, ncclFloat64, ncclSum, c->comm, s));
        NCCL_TRY(ncclAllReduce(c->scal_d, c->scal_d, 1, ncclInt32, ncclSum, c->comm, s));
        // the error word (label out of range, halo overflow, barrier timeout) is max-reduced so
        // every rank skips the update below and reports the error (no rank runs on alone)
        NCCL_TRY(ncclAllReduce(c->scal_d + 1, c->scal_d + 1, 1, ncclInt32, ncclMax, c->comm, s));
        NCCL_TRY(ncclGroupEnd());
    }
    c->step_t++;
    const double bc1 = 1.0 - std::pow(c->cfg.beta1, (double)c->step_t);
    const double bc2 = 1.0 - std::pow(c->cfg.beta2, (double)c->step_t);
    for (int l = 1; l <= L; ++l) {
        const int64_t off = c->woff[l - 1], cnt = c->woff[l] - off;
        launch_optimizer(c->cfg.optimizer, W[l - 1], c->dW + off, c->adam_m + off, c->adam_v + off,
                         cnt, (float)c->cfg.lr, (float)c->cfg.beta1, (float)c->cfg.beta2,
                         (float)c->cfg.adam_eps, (float)bc1, (float)bc2, c->scal_d + 1, s);
        c->launches++;
    }
    CDF_TRY(check_launch("optimizer"));
    mark(c, PH_END, s);
    // ---- read back loss / accuracy / counters (C5) and update ε
    double* hd = c->host_scratch;
    CUDA_TRY(cudaMemcpyAsync(hd, c->loss_d, sizeof(double) * k, cudaMemcpyDeviceToHost, s));
    int32_t* hi = reinterpret_cast<int32_t*>(hd + k);
    CUDA_TRY(cudaMemcpyAsync(hi, c->scal_d, sizeof(int32_t) * 2, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(c->stats_h, c->stats_d, sizeof(long long) * L * 2 * 4, cudaMemcpyDeviceToHost, s));
    CDF_TRY(wait_stream(c, s));
    if (hi[1] != 0) {
        c->step_t--;                   // the optimizer skipped this epoch's update (W unchanged)
        if (hi[1] == 3) CDF_FAIL(CDFGNN_EDATA, "label out of range");
        CDF_FAIL(CDFGNN_EPROTO, "halo protocol violation (code %d)", hi[1]);
    }
    double loss = 0.0;
    for (int t = 0; t < k; ++t) loss += hd[t];
    loss /= (double)c->ntrain;
    const int64_t correct = hi[0];
    const double acc = (double)correct / (double)c->ntrain;
    if (out) {
        std::memset(out, 0, sizeof(*out));
        out->loss = loss;
        out->correct = correct;
        out->total = c->ntrain;
        out->acc = acc;
        out->eps_used = eps_used;
        for (int l = 1; l <= L; ++l)
            for (int dir = 0; dir < 2; ++dir)
                fill_sync_stats(c, l, dir, c->stats_h + ((l - 1) * 2 + dir) * 4, wire[l - 1][dir],
                                dir ? &out->bwd[l - 1] : &out->fwd[l - 1]);
        out->gpu_launches = c->launches;
        out->transport = c->transport;
        if (c->timing && c->ev_used >= 2) {
            double ph[5] = {0, 0, 0, 0, 0};
            std::vector<std::pair<int64_t, std::pair<int, double>>> per;   // ld -> (launches, ms)
            for (size_t e = 0; e + 1 < c->ev_used; ++e) {
                float ms = 0.f;
                cudaEventElapsedTime(&ms, c->ev[e], c->ev[e + 1]);
                ph[c->ev_phase[e]] += ms;
                if (c->ev_phase[e] == PH_SYNC && c->ev_tag[e] >= 0 && c->ev_tag[e] < 6)
                    out->ms_sync_sub[c->ev_tag[e]] += ms;
                if (c->ev_phase[e] == PH_SPMM) {
                    bool found = false;
                    for (auto& q : per)
                        if (q.first == c->ev_tag[e]) { q.second.first++; q.second.second += ms; found = true; }
                    if (!found) per.push_back({c->ev_tag[e], {1, (double)ms}});
                }
            }
            out->ms_gemm = ph[PH_GEMM];
            out->ms_spmm = ph[PH_SPMM];
            out->ms_sync = ph[PH_SYNC];
            out->ms_other = ph[PH_OTHER];
            size_t best = 0;
            for (size_t q = 1; q < per.size(); ++q)
                if (per[q].second.second > per[best].second.second) best = q;
            if (!per.empty()) {
                const double ld = (double)per[best].first;
                out->spmm_ld = (int32_t)per[best].first;
                out->spmm_launches = per[best].second.first;
                out->spmm_ms_sum = per[best].second.second;
                // every part launches each width once per direction: bytes per launch averaged
                double g = 0, cpl = 0;
                for (const LocalPart& P : c->parts) {
                    g += 4.0 * (P.n + 1) + 8.0 * P.nnz + 4.0 * ld * P.nnz + 4.0 * ld * P.n;
                    cpl += 4.0 * (P.n + 1) + 8.0 * P.nnz + 4.0 * ld * P.n + 4.0 * ld * P.n;
                }
                const double per_launch = g / c->k, per_launch_c = cpl / c->k;
                out->spmm_bytes = per_launch * out->spmm_launches;
                out->spmm_bytes_compulsory = per_launch_c * out->spmm_launches;
            }
        }
    }
    // ε controller (R17, R18): first epoch seeds mean_acc without changing ε
    if (!c->have_mean) {
        c->mean_acc = acc;
        c->have_mean = true;
    } else {
        if (c->cfg.adaptive) c->eps = update_eps(c->cfg, c->eps, acc, c->mean_acc);
        c->mean_acc = 0.8 * c->mean_acc + 0.2 * acc;
    }
    if (out) out->eps_next = c->cfg.cache_on ? c->eps : 0.0;
    return CDFGNN_OK;
}

extern "C" int cdfgnn_epoch(cdfgnn_ctx* c, const float* const* X, const int32_t* const* labels,
                            const uint8_t* const* train_mask, float* const* W,
                            cdfgnn_epoch_stats* out, void* stream) {
    if (!c || !X || !labels || !train_mask || !W) CDF_FAIL(CDFGNN_EUSAGE, "NULL argument");
    CUDA_TRY(cudaSetDevice(c->device));
    c->in_epoch = true;
    const int rc = epoch_impl(c, X, labels, train_mask, W, out, (cudaStream_t)stream);
    c->in_epoch = false;
    return rc;
}

namespace {
void stage_slot(LocalPart& P, int slot, float** X, int32_t** lab, uint8_t** msk) {
    *X = slot ? P.X_stage1 : P.X_stage;
    *lab = slot ? P.lab_stage1 : P.lab_stage;
    *msk = slot ? P.mask_stage1 : P.mask_stage;
}
int copy_inputs(cdfgnn_ctx* c, int slot, const float* const* X_host, const int32_t* const* labels_host,
                const uint8_t* const* mask_host, cudaStream_t s) {
    const int64_t ld0 = ld_of(c->cfg.dims[0]);
    for (int t = 0; t < c->k; ++t) {
        LocalPart& P = c->parts[t];
        float* X; int32_t* lab; uint8_t* msk;
        stage_slot(P, slot, &X, &lab, &msk);
        // new contents in a library-owned staging buffer: the per-X-buffer caches of
        // static_inputs (Â_i X_i, Xᵀ) keyed on its pointer are stale
        if (P.ax_src == X) P.ax_src = nullptr;
        if (P.xT_src == X) P.xT_src = nullptr;
        if (c->comm_in) {
            // owned rows only (boundary masters [0, B), interior [B + M, n)); the M mirror rows
            // are replicas of other parts' masters and arrive from them below
            CUDA_TRY(cudaMemcpyAsync(X, X_host[t], sizeof(float) * P.B * ld0, cudaMemcpyHostToDevice, s));
            const int64_t i0 = P.B + P.M;
            CUDA_TRY(cudaMemcpyAsync(X + i0 * ld0, X_host[t] + i0 * ld0, sizeof(float) * (P.n - i0) * ld0,
                                     cudaMemcpyHostToDevice, s));
        } else {
            CUDA_TRY(cudaMemcpyAsync(X, X_host[t], sizeof(float) * P.n * ld0, cudaMemcpyHostToDevice, s));
        }
        CUDA_TRY(cudaMemcpyAsync(lab, labels_host[t], sizeof(int32_t) * P.n, cudaMemcpyHostToDevice, s));
        CUDA_TRY(cudaMemcpyAsync(msk, mask_host[t], P.n, cudaMemcpyHostToDevice, s));
        if (c->comm_in) {
            // masters' rows for every mirror peer q (halo list order = q's mirror slab order, R21)
            const int p = c->p, me = P.part;
            c->launches += launch_gather_rows(X, ld0, P.halo_local, P.hoff[p], P.xpack, s);
            CDF_TRY(check_launch("gather_rows"));
            NCCL_TRY(ncclGroupStart());
            for (int q = 0; q < p; ++q) {
                if (q == me) continue;
                if (P.capB[q] > 0)
                    NCCL_TRY(ncclSend(P.xpack + P.hoff[q] * ld0, (size_t)(P.capB[q] * ld0), ncclFloat32, q,
                                      c->comm_in, s));
                if (P.capA[q] > 0)
                    NCCL_TRY(ncclRecv(X + (P.B + P.moff[q]) * ld0, (size_t)(P.capA[q] * ld0), ncclFloat32, q,
                                      c->comm_in, s));
            }
            NCCL_TRY(ncclGroupEnd());
        }
    }
    return CDFGNN_OK;
}
}  // namespace

extern "C" int cdfgnn_epoch_host_next(cdfgnn_ctx* c, const float* const* X_host,
                                      const int32_t* const* labels_host,
                                      const uint8_t* const* train_mask_host,
                                      const float* const* X_next, const int32_t* const* labels_next,
                                      const uint8_t* const* train_mask_next, float* const* W,
                                      cdfgnn_epoch_stats* out, void* stream) {
    if (!c || !W) CDF_FAIL(CDFGNN_EUSAGE, "NULL argument");
    if ((X_next != nullptr) != (labels_next != nullptr) || (X_next != nullptr) != (train_mask_next != nullptr))
        CDF_FAIL(CDFGNN_EUSAGE, "X_next, labels_next and train_mask_next must be all set or all NULL");
    CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = (cudaStream_t)stream;
    if (!c->cs) {
        CUDA_TRY(cudaStreamCreateWithFlags(&c->cs, cudaStreamNonBlocking));
        for (int i = 0; i < 2; ++i) {
            CUDA_TRY(cudaEventCreateWithFlags(&c->staged[i], cudaEventDisableTiming));
            CUDA_TRY(cudaEventCreateWithFlags(&c->used[i], cudaEventDisableTiming));
            CUDA_TRY(cudaEventRecord(c->used[i], c->cs));
        }
    }
    int cur = c->prefetched;
    if (cur >= 0) {
        CUDA_TRY(cudaStreamWaitEvent(s, c->staged[cur], 0));     // this step's inputs, copied under the last step
    } else {
        if (!X_host || !labels_host || !train_mask_host) CDF_FAIL(CDFGNN_EUSAGE, "NULL argument");
        cur = 0;
        // on the copy stream (the only stream that issues comm_in operations), then joined
        CUDA_TRY(cudaEventRecord(c->staged[1], s));
        CUDA_TRY(cudaStreamWaitEvent(c->cs, c->staged[1], 0));
        CUDA_TRY(cudaStreamWaitEvent(c->cs, c->used[0], 0));
        CDF_TRY(copy_inputs(c, 0, X_host, labels_host, train_mask_host, c->cs));
        CUDA_TRY(cudaEventRecord(c->staged[0], c->cs));
        CUDA_TRY(cudaStreamWaitEvent(s, c->staged[0], 0));
    }
    c->prefetched = -1;
    if (X_next) {
        // the next step's inputs go to the other slot on the copy stream, overlapping this epoch
        const int nxt = 1 - cur;
        CUDA_TRY(cudaStreamWaitEvent(c->cs, c->used[nxt], 0));
        CDF_TRY(copy_inputs(c, nxt, X_next, labels_next, train_mask_next, c->cs));
        CUDA_TRY(cudaEventRecord(c->staged[nxt], c->cs));
        c->prefetched = nxt;
    }
    std::vector<const float*> X(c->k);
    std::vector<const int32_t*> lab(c->k);
    std::vector<const uint8_t*> msk(c->k);
    for (int t = 0; t < c->k; ++t) {
        float* x; int32_t* l; uint8_t* m;
        stage_slot(c->parts[t], cur, &x, &l, &m);
        X[t] = x; lab[t] = l; msk[t] = m;
    }
    c->in_epoch = true;
    const int rc = epoch_impl(c, X.data(), lab.data(), msk.data(), W, out, s);
    c->in_epoch = false;
    cudaEventRecord(c->used[cur], s);
    return rc;
}

extern "C" int cdfgnn_epoch_host(cdfgnn_ctx* c, const float* const* X_host,
                                 const int32_t* const* labels_host,
                                 const uint8_t* const* train_mask_host, float* const* W,
                                 cdfgnn_epoch_stats* out, void* stream) {
    if (!c || !X_host || !labels_host || !train_mask_host || !W) CDF_FAIL(CDFGNN_EUSAGE, "NULL argument");
    CUDA_TRY(cudaSetDevice(c->device));
    cudaStream_t s = (cudaStream_t)stream;
    if (c->prefetched >= 0) {           // a prefetch from cdfgnn_epoch_host_next is discarded
        CUDA_TRY(cudaStreamWaitEvent(s, c->staged[c->prefetched], 0));
        c->prefetched = -1;
    }
    if (c->cs) CUDA_TRY(cudaStreamWaitEvent(s, c->used[0], 0));
    const int64_t ld0 = ld_of(c->cfg.dims[0]);
    std::vector<const float*> X(c->k);
    std::vector<const int32_t*> lab(c->k);
    std::vector<const uint8_t*> msk(c->k);
    for (int t = 0; t < c->k; ++t) {
        LocalPart& P = c->parts[t];
        if (P.ax_src == P.X_stage) P.ax_src = nullptr;     // staging rewritten: static-input caches stale
        if (P.xT_src == P.X_stage) P.xT_src = nullptr;
        CUDA_TRY(cudaMemcpyAsync(P.X_stage, X_host[t], sizeof(float) * P.n * ld0, cudaMemcpyHostToDevice, s));
        CUDA_TRY(cudaMemcpyAsync(P.lab_stage, labels_host[t], sizeof(int32_t) * P.n, cudaMemcpyHostToDevice, s));
        CUDA_TRY(cudaMemcpyAsync(P.mask_stage, train_mask_host[t], P.n, cudaMemcpyHostToDevice, s));
        X[t] = P.X_stage; lab[t] = P.lab_stage; msk[t] = P.mask_stage;
    }
    c->in_epoch = true;
    const int rc = epoch_impl(c, X.data(), lab.data(), msk.data(), W, out, s);
    c->in_epoch = false;
    return rc;
}

extern "C" int cdfgnn_cache_view(cdfgnn_ctx* c, int32_t lp, int32_t l, int32_t dir, int32_t which,
                                 float** ptr, int64_t* rows, int64_t* ld) {
    if (!c || !ptr || !rows || !ld) CDF_FAIL(CDFGNN_EUSAGE, "NULL argument");
    if (lp < 0 || lp >= c->k || l < 1 || l > c->cfg.L || dir < 0 || dir > 1)
        CDF_FAIL(CDFGNN_EUSAGE, "bad part/layer/dir");
    if (!c->cfg.cache_on) CDF_FAIL(CDFGNN_EUSAGE, "cache is off");
    const LocalPart& P = c->parts[lp];
    const CacheDev& cd = P.cache[l - 1][dir];
    *ld = ld_of(c->cfg.dims[l]);
    switch (which) {
        case 0: *ptr = cd.s_mir; *rows = P.M; break;
        case 1: *ptr = cd.b_mir; *rows = P.M; break;
        case 2: *ptr = cd.s_mas; *rows = P.B; break;
        case 3: *ptr = cd.a; *rows = P.B; break;
        case 4: *ptr = cd.b_mas; *rows = P.B; break;
        default: CDF_FAIL(CDFGNN_EUSAGE, "which must be 0..4");
    }
    return CDFGNN_OK;
}

extern "C" int cdfgnn_act_view(cdfgnn_ctx* c, int32_t lp, int32_t l, float** ptr, int64_t* rows, int64_t* ld) {
    if (!c || !ptr || !rows || !ld) CDF_FAIL(CDFGNN_EUSAGE, "NULL argument");
    if (lp < 0 || lp >= c->k || l < 1 || l > c->cfg.L) CDF_FAIL(CDFGNN_EUSAGE, "bad part/layer");
    const LocalPart& P = c->parts[lp];
    *ptr = P.act[l];
    *rows = P.n;
    *ld = ld_of(c->cfg.dims[l]);
    return CDFGNN_OK;
}

extern "C" int cdfgnn_grad_view(cdfgnn_ctx* c, int32_t l, float** ptr, int64_t* rows, int64_t* ld) {
    if (!c || !ptr || !rows || !ld) CDF_FAIL(CDFGNN_EUSAGE, "NULL argument");
    if (l < 1 || l > c->cfg.L) CDF_FAIL(CDFGNN_EUSAGE, "bad layer");
    *ptr = c->dW + c->woff[l - 1];
    *rows = c->cfg.dims[l - 1];
    *ld = c->cfg.dims[l];
    return CDFGNN_OK;
}

extern "C" int cdfgnn_sync_flags(cdfgnn_ctx* c, int32_t lp, int32_t l, int32_t dir, int32_t which,
                                 uint8_t** ptr, int64_t* rows) {
    if (!c || !ptr || !rows) CDF_FAIL(CDFGNN_EUSAGE, "NULL argument");
    if (lp < 0 || lp >= c->k) CDF_FAIL(CDFGNN_EUSAGE, "bad part");
    if (l < 1 || l > c->cfg.L || dir < 0 || dir > 1) CDF_FAIL(CDFGNN_EUSAGE, "bad layer/dir");
    const LocalPart& P = c->parts[lp];
    const HaloDev h = halo_for(c, P, l, dir);
    switch (which) {
        case 0: *ptr = h.gflag; *rows = P.M; break;
        case 1: *ptr = h.fired; *rows = P.B; break;
        case 2: *ptr = h.active; *rows = P.B; break;
        default: CDF_FAIL(CDFGNN_EUSAGE, "which must be 0..2");
    }
    return CDFGNN_OK;
}

extern "C" int cdfgnn_msg_view(cdfgnn_ctx* c, int32_t lp, int32_t phase, int32_t src, cdfgnn_msg_view_t* out) {
    if (!c || !out) CDF_FAIL(CDFGNN_EUSAGE, "NULL argument");
    if (lp < 0 || lp >= c->k || phase < 0 || phase > 1 || src < 0 || src >= c->p)
        CDF_FAIL(CDFGNN_EUSAGE, "bad part/phase/source");
    const LocalPart& P = c->parts[lp];
    if (src == P.part) CDF_FAIL(CDFGNN_EUSAGE, "a part sends no messages to itself");
    std::memset(out, 0, sizeof(*out));
    const int bits = c->cfg.quant_bits;
    const int64_t ld = c->last_ld[phase] ? c->last_ld[phase] : c->ldmax;
    out->quant_bits = bits;
    out->row_bytes = code_row_bytes(bits, ld);
    // gather messages at the master are indexed by the halo list (src -> me), scatter messages
    // at the mirror by the mirror slab of master src (the same list seen from the other side)
    out->capacity = phase == 0 ? P.capB[src] : P.capA[src];
    if (c->slot) {
        out->layout = 1;
        out->base = phase == 0 ? P.gsrc.base[src] : P.ssrc.base[src];
        out->hdr_bytes = 16;
        out->slot_bytes = slot_stride(bits, ld);
        out->stamp = c->last_stamp[phase];
    } else {
        const RegionTab& rt = phase == 0 ? P.grecv_h : P.srecv_h;
        out->layout = 0;
        out->base = rt.hdr[src];
        out->pay = rt.pay[src];
        out->count = rt.cnt[src];
        out->hdr_bytes = c->hdr_bytes;
    }
    return CDFGNN_OK;
}

extern "C" int cdfgnn_reset_caches(cdfgnn_ctx* c, void* stream) {
    if (!c) CDF_FAIL(CDFGNN_EUSAGE, "NULL ctx");
    cudaStream_t s = (cudaStream_t)stream;
    CUDA_TRY(cudaSetDevice(c->device));
    for (LocalPart& P : c->parts)
        for (int l = 1; l <= c->cfg.L; ++l) {
            const int64_t ld = ld_of(c->cfg.dims[l]);
            for (int dir = 0; dir < 2; ++dir) {
                CacheDev& cd = P.cache[l - 1][dir];
                if (!cd.s_mir) continue;
                CUDA_TRY(cudaMemsetAsync(cd.s_mir, 0, sizeof(float) * P.M * ld, s));
                CUDA_TRY(cudaMemsetAsync(cd.b_mir, 0, sizeof(float) * P.M * ld, s));
                CUDA_TRY(cudaMemsetAsync(cd.s_mas, 0, sizeof(float) * P.B * ld, s));
                CUDA_TRY(cudaMemsetAsync(cd.a, 0, sizeof(float) * P.B * ld, s));
                CUDA_TRY(cudaMemsetAsync(cd.b_mas, 0, sizeof(float) * P.B * ld, s));
            }
        }
    return CDFGNN_OK;
}

extern "C" int cdfgnn_get_eps(cdfgnn_ctx* c, double* eps, double* mean_acc) {
    if (!c) CDF_FAIL(CDFGNN_EUSAGE, "NULL ctx");
    if (eps) *eps = c->eps;
    if (mean_acc) *mean_acc = c->mean_acc;
    return CDFGNN_OK;
}

extern "C" int cdfgnn_set_eps(cdfgnn_ctx* c, double eps) {
    if (!c) CDF_FAIL(CDFGNN_EUSAGE, "NULL ctx");
    if (!(eps >= 0.0)) CDF_FAIL(CDFGNN_EUSAGE, "eps must be >= 0");
    c->eps = eps;
    return CDFGNN_OK;
}

extern "C" int cdfgnn_spmm(cdfgnn_ctx* c, int32_t lp, const float* T, float* Y, int64_t ld, int32_t F,
                           void* stream) {
    if (!c || !T || !Y) CDF_FAIL(CDFGNN_EUSAGE, "NULL argument");
    if (lp < 0 || lp >= c->k) CDF_FAIL(CDFGNN_EUSAGE, "bad part");
    if (ld % 4 || ld < F || ld > 1024) CDF_FAIL(CDFGNN_EUSAGE, "ld must be a multiple of 4 in [F, 1024]");
    CUDA_TRY(cudaSetDevice(c->device));
    LocalPart& P = c->parts[lp];
    const SpmmPlan& S = spmm_plan(P, ld);
    if (S.nslots && ld > S.pstride)
        CDF_FAIL(CDFGNN_EUSAGE, "ld %lld exceeds the split-row scratch stride %lld (widest layer)", (long long)ld,
                 (long long)S.pstride);
    (void)S;
    return spmm_part(c, P, T, Y, ld, (cudaStream_t)stream, 0);
}

extern "C" int cdfgnn_bandwidth_probe(const void* buf, int64_t bytes, int32_t reps, double* gbs, void* stream) {
    if (!buf || !gbs || bytes < 16 || reps < 1) CDF_FAIL(CDFGNN_EUSAGE, "bad probe arguments");
    cudaStream_t s = (cudaStream_t)stream;
    const float4* p = reinterpret_cast<const float4*>(buf);
    const int64_t n4 = bytes / 16;
    launch_read_probe(p, n4, 1, nullptr, s);    // warm (L2-resident for small buffers)
    cudaEvent_t e0, e1;
    CUDA_TRY(cudaEventCreate(&e0));
    CUDA_TRY(cudaEventCreate(&e1));
    CUDA_TRY(cudaEventRecord(e0, s));
    launch_read_probe(p, n4, reps, nullptr, s);
    CUDA_TRY(cudaEventRecord(e1, s));
    CUDA_TRY(cudaEventSynchronize(e1));
    float ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *gbs = (double)n4 * 16.0 * reps / (ms * 1e-3) / 1e9;
    return check_launch("probe");
}

extern "C" const char* cdfgnn_last_error(void) { return cdfgnn::g_err.c_str(); }
extern "C" const char* cdfgnn_version(void) { return "cdfgnn-b200 0.1 (sm_100a)"; }
