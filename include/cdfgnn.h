/*
 * cdfgnn.h — C ABI of the B200-native CDFGNN hot path (arXiv 2408.00232).
 *
 * One call per step of the paper's per-layer distributed full-batch GCN
 * iteration (Alg. 1):
 *
 *   cdfgnn_partition      hierarchical EBV vertex-cut (§6), host
 *   cdfgnn_layer_fwd      Z̈_i = Â_i H_i W (eq. 1) → sync → H = σ(Z)
 *   cdfgnn_layer_bwd      sync δ̈ → δ; ∇W = Hᵀ Â_i δ (eq. 5);
 *                         δ̈^(l-1) = (Â_i δ Wᵀ) ⊙ σ'(Z^(l-1))
 *   cdfgnn_halo_exchange  one gather + scatter synchronisation (§3.2)
 *                         with the adaptive vertex cache (Alg. 2) and
 *                         B-bit linear quantisation (§5)
 *   cdfgnn_epoch          Alg. 1 end to end, incl. loss on masters,
 *                         parameter aggregation and the ε
 *                         controller
 *
 * Conventions
 *  - All functions return a status code (CDFGNN_OK = 0); on failure
 *    cdfgnn_last_error() returns a thread-local message.  No C++ exception
 *    crosses the ABI.
 *  - Host pointers are plain host memory; "device" pointers are CUDA device
 *    memory of the context's device.  Every device pointer the caller passes
 *    is caller-owned, 16-byte aligned, row-major with a leading dimension
 *    ld % 4 == 0 whose padding columns are zero (reading R24).
 *  - Device memory is owned by the caller: the context carves every buffer
 *    (CSR copies, caches, message staging, activations) out of one caller
 *    allocated workspace (cdfgnn_workspace_size / cdfgnn_init).  The library
 *    owns only the context object and its NCCL communicator.
 *  - `stream` is a cudaStream_t passed as void*.  Calls are asynchronous on it
 *    except where a function says it synchronises (NCCL message counts need a
 *    device→host read, see cdfgnn_halo_exchange).
 *  - Vertex ids are int32 (n < 2^31).  Local row order of a part (reading R21):
 *    [boundary masters ↑gid][mirrors grouped by master part ↑, then ↑gid]
 *    [interior ↑gid].
 *  Readings R1..R27 are listed in DESIGN.md §"Readings of the paper".
 */
#ifndef CDFGNN_H
#define CDFGNN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (codes 0/2/3/4 align with SPEC S:L648) */
#define CDFGNN_OK 0
#define CDFGNN_EUSAGE 2      /* bad argument / shape / call order */
#define CDFGNN_EDATA 3       /* invalid input data (edge out of range, duplicate, label >= C) */
#define CDFGNN_EPROTO 4      /* protocol / internal invariant violated */
#define CDFGNN_ECUDA 5       /* CUDA runtime error */
#define CDFGNN_ENCCL 6       /* NCCL error */
#define CDFGNN_EWORKSPACE 7  /* workspace too small */

#define CDFGNN_MAX_PARTS 64
#define CDFGNN_MAX_LAYERS 8

typedef struct cdfgnn_plan cdfgnn_plan;
typedef struct cdfgnn_ctx cdfgnn_ctx;

/* ------------------------------------------------------------------------- */
/* Partitioning (host).  Eq. Eva:                                 */
/*   Eva_(u,v)(i) = (1-γ)(𝟙[i∉d_rep_u] + 𝟙[i∉d_rep_v])                         */
/*                + γ(𝟙[host_i∉h_rep_u] + 𝟙[host_i∉h_rep_v])                   */
/*                + α e_count[i]/(|E|/p) + β v_count[i]/(|V|/p)               */
/* evaluated exactly (integer scaled), argmin with ties to the lowest part id. */
/* ------------------------------------------------------------------------- */
typedef struct {
    int32_t num_parts;          /* p, 1..64 */
    int32_t num_hosts;          /* 1 on a single box (reading R22) */
    const int32_t* host_of;     /* [p] part -> host, or NULL: host = i*num_hosts/p */
    int64_t alpha_num, alpha_den;   /* α (default 1/1) */
    int64_t beta_num, beta_den;     /* β (default 1/1) */
    int64_t gamma_num, gamma_den;   /* γ (default 1/10) */
    int32_t edge_order;         /* 0 input order, 1 ascending (d_u+d_v) then (min,max) id
                                   (default, reading R19), 2 splitmix64 shuffle by seed */
    uint64_t seed;
    int32_t self_loops;         /* 0 = literal Â (reading R1); 1 = A + I, loop in the master's part */
} cdfgnn_partition_cfg;

typedef struct {
    int32_t part;
    int64_t n_local;            /* |V_i| */
    int64_t n_bmaster;          /* B_i: boundary masters (rows [0, B_i)) */
    int64_t n_mirror;           /* M_i: mirrors (rows [B_i, B_i+M_i)) */
    int64_t n_edges;            /* |E_i| undirected edges assigned to the part */
    int64_t nnz;                /* CSR entries of Â_i */
    const int32_t* local2global;    /* [n_local] */
    const int32_t* rowptr;          /* [n_local+1] */
    const int32_t* colidx;          /* [nnz], ascending within a row */
    const float* val;               /* [nnz], 1/sqrt(d_u d_v), global degrees (R2) */
    const int64_t* mirror_off;      /* [p+1]: mirrors of master part j are rows
                                       [B_i+mirror_off[j], B_i+mirror_off[j+1]) */
    const int64_t* halo_off;        /* [p+1]: halo list (s -> this part) occupies
                                       halo_local[halo_off[s] .. halo_off[s+1]) */
    const int32_t* halo_local;      /* local master rows of each halo list, in list order
                                       (list (s,i) = vertices mastered here with a mirror on s,
                                       ascending global id) */
} cdfgnn_part_view;

typedef struct {
    double rf;                  /* Σ|V_i| / |V| */
    double edge_if;             /* max|E_i| / (|E|/p) */
    double vertex_if;           /* max|V_i| / (Σ|V_i|/p) */
    int64_t total_mirrors;      /* M = Σ_u (r_u - 1) */
    int64_t inner_max;          /* Table 3 "Inner" */
    int64_t outer_max;          /* Table 3 "Outer" */
    int64_t sum_vi;
    int64_t max_ei;
} cdfgnn_partition_stats;

/* Fill cfg with the defaults above for p parts. */
int cdfgnn_partition_cfg_default(cdfgnn_partition_cfg* cfg, int32_t p);

/* Partition m undirected edges (stored once, no duplicates, no self-loops, ids < n).
 * edge_part [m] and master [n] are caller-owned outputs (may be NULL).
 * *plan is library-owned; free with cdfgnn_plan_free.
 * Errors: p < 1 or p > 64 or m == 0 -> EUSAGE; endpoint >= n, self-loop or
 * duplicate edge -> EDATA.  Deterministic for fixed inputs. */
int cdfgnn_partition(int64_t n, int64_t m, const int32_t* eu, const int32_t* ev,
                     const cdfgnn_partition_cfg* cfg, int32_t* edge_part, int32_t* master,
                     cdfgnn_plan** plan);
int cdfgnn_plan_num_parts(const cdfgnn_plan* plan);
/* Borrowed view of one part, valid until cdfgnn_plan_free. */
int cdfgnn_plan_part(const cdfgnn_plan* plan, int32_t part, cdfgnn_part_view* out);
int cdfgnn_plan_stats(const cdfgnn_plan* plan, cdfgnn_partition_stats* out);
void cdfgnn_plan_free(cdfgnn_plan* plan);

/* ------------------------------------------------------------------------- */
/* Training context                                                          */
/* ------------------------------------------------------------------------- */
typedef struct {
    int32_t L;                          /* layers */
    int32_t dims[CDFGNN_MAX_LAYERS + 1];/* F_0 .. F_L */
    int32_t cache_on;                   /* 1: Alg. 2 cache; 0: no-cache baseline (reading R14) */
    double eps_init;                    /* ε₀ (reading R18: 0.01) */
    int32_t adaptive;                   /* 1: ε controller P:L386-399 */
    double mu1, mu2, nu1, nu2, xi, lam1, lam2;  /* P:L399 defaults */
    int32_t eps_clamp;                  /* 1: clamp ε to [ν2, ν1] (reading R17) */
    int32_t quant_bits;                 /* B of §5 (B is left free by the paper):
                                           0 = fp32 payloads; 4, 8 (default) or 16-bit codes
                                           (reading R15; code rows: B = 8 one byte per code,
                                           B = 4 two per byte — code k in the low nibble of byte
                                           k/2 for even k —, B = 16 little-endian uint16) */
    int32_t optimizer;                  /* 0 SGD, 1 Adam */
    double lr, beta1, beta2, adam_eps;
    int32_t gemm_tf32;                  /* 3: tcgen05 3xTF32 GEMMs (default, ~fp32 accuracy);
                                           1: tcgen05 1xTF32; 0: fp32 SIMT GEMMs */
    int32_t timing;                     /* 1: per-phase CUDA-event timing in epoch stats */
    int32_t transport;                  /* world > 1: 0 = NVLink push (pack kernels store into
                                           peers' receive regions through CUDA IPC mappings,
                                           one NCCL barrier per phase, no host round trip;
                                           falls back to 1 if IPC is unavailable);
                                           1 = NCCL grouped send/recv after a count exchange */
    int32_t elide_dead_syncs;           /* 1 (default): inside cdfgnn_epoch skip the layer-L forward
                                           scatter and backward gather (§8 f2; bitwise-identical
                                           results: mirrors never read logits and their δ̈^(L) = 0) */
    int32_t static_inputs;              /* 1: the input features X do not change between calls for
                                           a given buffer, so Xᵀ (∇W^(0) operand) is built once per
                                           X pointer and reused; 0 (default): rebuilt every epoch;
                                           2: also hoist the layer-1 aggregation — Â_i X_i is built
                                           once per X pointer, layer 1 runs (Â_i X_i) W^(0) and
                                           ∇W^(0) = (Â_i X_i)ᵀ δ^(1) (associativity of eq. (1),
                                           P:L236-238, and of P:L273-278 with Â_i symmetric): both
                                           layer-1 SpMMs leave the epoch; results equal the
                                           per-epoch schedule up to fp32 rounding order */
    int32_t overlap;                    /* 1: boundary-rows-first scheduling (§8 f1) — the SpMM
                                           (forward) or ∇H GEMM (backward, inside cdfgnn_epoch)
                                           produces the mirror rows first, their gather phase (test,
                                           pack, NVLink push, barrier) runs on a second, high-priority
                                           stream while the master and interior rows are computed.
                                           Bitwise-identical results; used when p > 1 and the
                                           transport has no host round trip (push or co-resident).
                                           0 (default): measured slower on B200 — the
                                           split SpMM and the concurrent streaming kernels cost more
                                           L2 bandwidth than the hidden gather saves */
    int32_t msg_layout;                 /* message regions: 0 (default) = slot-addressed for
                                           co-resident parts and the NVLink push transport,
                                           compacted for NCCL send/recv; 1 = compacted always
                                           (per-peer packed buffers: ballot + prefix compaction,
                                           counts, index maps, a copy kernel for push);
                                           2 = slot-addressed (EUSAGE with transport = 1).
                                           Slot-addressed: the message of the vertex at
                                           halo-list position k lives in slot k of the (source,
                                           destination) region — header {u32 stamp, f32 lo,
                                           f32 hi, u32 0} + code row — stamped with the phase's
                                           sequence number; senders store straight into the
                                           receiver's region (through CUDA IPC on a peer GPU) */
    int32_t fuse_gather;                /* 1 (default): with the slot layout and p > 1 the forward
                                           SpMM's epilogue runs the gather of its synchronisation
                                           (Alg. 2 L3-L9: test, quantise, slot store, snapshot) on the
                                           mirror rows it just computed, from registers (§8 f1);
                                           0: separate gather kernel.  Bitwise-identical results */
} cdfgnn_cfg;

int cdfgnn_cfg_default(cdfgnn_cfg* cfg);

/* 128-byte NCCL unique id (rank 0 creates it, the caller broadcasts it). */
int cdfgnn_get_unique_id(void* out128);

/* Bytes of device workspace a context for the k local parts `parts` needs.
 * world > 1 requires k == 1 (one partition per GPU); world == 1 may host all p
 * parts (co-resident partitions exchange through device memory). */
int cdfgnn_workspace_size(const cdfgnn_plan* plan, const int32_t* parts, int32_t k,
                          const cdfgnn_cfg* cfg, size_t* bytes);

/* Create a context on `device` over the caller's workspace (>= workspace_size
 * bytes, 256-byte aligned).  Copies the parts' CSR and halo lists to the device.
 * world > 1: joins an NCCL communicator of `world` ranks with nccl_uid. */
int cdfgnn_init(const cdfgnn_plan* plan, const int32_t* parts, int32_t k, int32_t rank,
                int32_t world, const void* nccl_uid, int32_t device, void* workspace,
                size_t workspace_bytes, const cdfgnn_cfg* cfg, cdfgnn_ctx** out);
int cdfgnn_destroy(cdfgnn_ctx* ctx);

/* Per-synchronisation counters (reading R25). */
typedef struct {
    int64_t gather_sent;        /* mirror -> master messages */
    int64_t master_fired;       /* masters whose own test fired (Alg. 2 L15) */
    int64_t active;             /* active masters (Alg. 2 L12, L18) */
    int64_t scatter_msgs;       /* master -> mirror messages */
    int64_t baseline;           /* 2 M: messages without the cache */
    int64_t bytes_alg;          /* ceil(B·F/8) + 12 per B-bit message (F+12 at B = 8: codes,
                                   lo, hi and a 32-bit position), 4F+4 per fp32 message */
    int64_t bytes_wire;         /* bytes that crossed to another GPU (NCCL payloads or
                                   NVLink stores: 16-byte header + code row per message in the
                                   slot layout); 0 for co-resident partitions */
} cdfgnn_sync_stats;

/* One gather + scatter synchronisation of layer l (1..L), direction dir
 * (0 = forward Z, 1 = backward δ) over the context's local parts.
 * X[k] (device, n_i x ld): in = local partials Z̈_i / δ̈_i; out = synced rows
 * (boundary rows from the cached aggregate; interior rows untouched).
 * eps: cache threshold (ignored with cache_on = 0).  st (host, may be NULL):
 * counters of this call — non-NULL forces a stream synchronisation.
 * Host synchronisation: none with the slot layout (co-resident parts, NVLink push: the
 * transfer barrier is a stream-ordered NCCL all-reduce); with the NCCL send/recv transport
 * the call synchronises `stream` twice (message counts).
 * Errors: l/dir/ld out of range -> EUSAGE; message count above the halo capacity or an
 * unknown position (compacted layout) -> EPROTO; NCCL failure -> ENCCL. */
int cdfgnn_halo_exchange(cdfgnn_ctx* ctx, int32_t l, int32_t dir, float* const* X, int64_t ld,
                         float eps, cdfgnn_sync_stats* st, void* stream);

/* Forward layer l: T = H_in W (W device [F_{l-1} x F_l] row-major), Z = Â_i T,
 * halo exchange on Z, H_out = ReLU(Z) (H_out may equal Z; NULL skips σ, as at l = L). */
int cdfgnn_layer_fwd(cdfgnn_ctx* ctx, int32_t l, const float* const* H_in, int64_t ld_in,
                     const float* W, float* const* Z, float* const* H_out, int64_t ld_out,
                     float eps, cdfgnn_sync_stats* st, void* stream);

/* Backward layer l: dZ[k] in = δ̈^(l), out = δ^(l) after the halo exchange;
 * S = Â_i δ; dW (device [F_{l-1} x F_l]) = Σ_local-parts H_inᵀ S (overwritten);
 * dZ_prev[k] (or NULL at l = 1) = (S Wᵀ) ⊙ 𝟙[H_in > 0]  (σ' of ReLU, R3). */
int cdfgnn_layer_bwd(cdfgnn_ctx* ctx, int32_t l, float* const* dZ, int64_t ld,
                     const float* const* H_in, int64_t ld_in, const float* W,
                     float* const* dZ_prev, float* dW, float eps, cdfgnn_sync_stats* st,
                     void* stream);

typedef struct {
    double loss;                /* mean CE over the global train set (reading R7) */
    int64_t correct, total;     /* train accuracy counts over masters (R16) */
    double acc;
    double eps_used, eps_next;
    cdfgnn_sync_stats fwd[CDFGNN_MAX_LAYERS];
    cdfgnn_sync_stats bwd[CDFGNN_MAX_LAYERS];
    int32_t gpu_launches;       /* kernels this library launched in the epoch */
    /* cfg.timing = 1: CUDA-event milliseconds per phase (summed over calls) */
    double ms_gemm, ms_spmm, ms_sync, ms_other;
    /* the dominant SpMM width (largest summed time) of this epoch: */
    int32_t spmm_ld;            /* its row width ld */
    int32_t spmm_launches;      /* its launches */
    double spmm_bytes;          /* their gather-model bytes */
    double spmm_bytes_compulsory;   /* their compulsory bytes */
    double spmm_ms_sum;         /* their summed CUDA-event time */
    double ms_sync_sub[6];      /* halo exchange split: gather pack, gather transfer, master apply,
                                   scatter pack, scatter transfer, mirror apply */
    int32_t transport;          /* 0 co-resident, 1 NCCL send/recv, 2 NVLink push */
} cdfgnn_epoch_stats;

/* Alg. 1 once.  X[k] device (n_i x ld(F_0)), labels[k] int32 [n_i],
 * train_mask[k] uint8 [n_i] (local row order), W[L] device, updated in place
 * (identical on every rank).  Synchronises `stream` at the end (loss/acc are
 * read back for the ε controller).  Label >= F_L -> EDATA. */
int cdfgnn_epoch(cdfgnn_ctx* ctx, const float* const* X, const int32_t* const* labels,
                 const uint8_t* const* train_mask, float* const* W, cdfgnn_epoch_stats* out,
                 void* stream);

/* Same, with X / labels / train_mask in HOST memory (pinned for best speed):
 * they are copied into context-owned device buffers inside the call. */
int cdfgnn_epoch_host(cdfgnn_ctx* ctx, const float* const* X_host,
                      const int32_t* const* labels_host, const uint8_t* const* train_mask_host,
                      float* const* W, cdfgnn_epoch_stats* out, void* stream);

/* Pipelined host inputs: runs Alg. 1 once on this step's host inputs and, when X_next /
 * labels_next / train_mask_next are non-NULL, starts copying the NEXT step's host inputs
 * into a second context-owned slot on an internal copy stream, overlapping this epoch.  On
 * the following call those prefetched inputs are used (its X_host/labels/mask arguments are
 * then ignored and may be NULL).  The *_next host buffers must stay unchanged until the next
 * call returns.  With one part per rank (world > 1) only the part's owned rows of X_host are
 * read — boundary masters [0, B) and interior rows [B + M, n); the M mirror rows are filled
 * from their masters' rows over NCCL (each vertex's features cross PCIe once), so mirror rows
 * of X_host need not be initialised.  Errors as cdfgnn_epoch; all three *_next set or all
 * NULL (else EUSAGE). */
int cdfgnn_epoch_host_next(cdfgnn_ctx* ctx, const float* const* X_host,
                           const int32_t* const* labels_host, const uint8_t* const* train_mask_host,
                           const float* const* X_next, const int32_t* const* labels_next,
                           const uint8_t* const* train_mask_next, float* const* W,
                           cdfgnn_epoch_stats* out, void* stream);

/* ---- introspection (tests, replay) ---- */
/* which: 0 mirror snapshot s, 1 mirror view b, 2 master snapshot s, 3 aggregate a,
 *        4 master view b.  Device pointer into the workspace. */
int cdfgnn_cache_view(cdfgnn_ctx* ctx, int32_t local_part, int32_t l, int32_t dir,
                      int32_t which, float** ptr, int64_t* rows, int64_t* ld);
/* Activations and parameter gradients of the most recent cdfgnn_epoch (device pointers into
 * the workspace, valid until the next call that runs layers):
 *   cdfgnn_act_view:  H^(l) = σ(Z^(l)) of local part `local_part` for l < L, the logits
 *                     Z^(L) for l = L (eqs. 1-2); rows = n_local, row stride ld(F_l),
 *                     local row order (R21).
 *   cdfgnn_grad_view: ∇W^(l-1) summed over all parts and ranks (Alg. 1 L12), the
 *                     value the optimizer consumed; [F_{l-1} x F_l] row-major (ld = F_l). */
int cdfgnn_act_view(cdfgnn_ctx* ctx, int32_t local_part, int32_t l, float** ptr, int64_t* rows, int64_t* ld);
int cdfgnn_grad_view(cdfgnn_ctx* ctx, int32_t l, float** ptr, int64_t* rows, int64_t* ld);
/* Cache-test decisions of the most recent synchronisation of layer l (1..L), direction dir
 * (0 = Z, 1 = δ) — the masks the oracle's follow mode replays.
 * which: 0 gather-sent flag per mirror row (Alg. 2 L4), 1 master-fired flag (L15), 2 active
 * flag (L12, L18).  uint8 per row, device pointer into the workspace.  A gather elided by
 * elide_dead_syncs leaves its flags 0 (no mirror sends). */
int cdfgnn_sync_flags(cdfgnn_ctx* ctx, int32_t local_part, int32_t l, int32_t dir, int32_t which,
                      uint8_t** ptr, int64_t* rows);

/* Messages received by local part `local_part` from part `src` in the most recent gather
 * (phase 0: mirror -> master, Alg. 2 L5-L8, at the master) or scatter (phase 1: master ->
 * mirror, L20-L22, at the mirror) phase (§5 message format).
 *  layout 1 (slot): base = region start; slot k (k < capacity, the halo-list length) at
 *    base + k*slot_bytes holds header {u32 stamp, f32 lo, f32 hi, u32 0} then row_bytes of
 *    codes (or the fp32 row); slot k carries a message of that phase iff its stamp == stamp.
 *  layout 0 (compacted): *count (device int32) messages; header k at hdr + k*hdr_bytes
 *    ({u32 halo-list position, f32 lo, f32 hi} or {u32 position}), row k at pay + k*row_bytes;
 *    order across blocks is not deterministic (the positions are).
 * Device pointers into the caller's workspace (or, co-resident, the sender's region), valid
 * until the next synchronisation; with one part per GPU the gather messages are valid only
 * until the same synchronisation's scatter (regions are reused).  row_bytes and stamp refer
 * to the width of that most recent phase. */
typedef struct {
    int32_t layout;             /* 0 compacted, 1 slot-addressed */
    const uint8_t* base;        /* slot: region start; compacted: header array */
    const uint8_t* pay;         /* compacted: payload rows; slot: NULL */
    const int32_t* count;       /* compacted: device message count; slot: NULL */
    int64_t capacity;           /* halo-list length of the (src, local part) pair */
    int64_t hdr_bytes;          /* 16 (slot), 12 or 4 (compacted) */
    int64_t row_bytes;          /* code / payload row bytes of the most recent phase */
    int64_t slot_bytes;         /* slot stride (slot layout) */
    uint32_t stamp;             /* slot layout: stamp of the most recent phase */
    int32_t quant_bits;
} cdfgnn_msg_view_t;
int cdfgnn_msg_view(cdfgnn_ctx* ctx, int32_t local_part, int32_t phase, int32_t src,
                    cdfgnn_msg_view_t* out);
int cdfgnn_reset_caches(cdfgnn_ctx* ctx, void* stream);
int cdfgnn_get_eps(cdfgnn_ctx* ctx, double* eps, double* mean_acc);
int cdfgnn_set_eps(cdfgnn_ctx* ctx, double eps);

/* Standalone local SpMM Y = Â_i T of local part `local_part` (a2), for the
 * roofline measurement; T, Y device (n_i x ld). */
int cdfgnn_spmm(cdfgnn_ctx* ctx, int32_t local_part, const float* T, float* Y, int64_t ld,
                int32_t F, void* stream);

/* Measurement helper (bench.py roofline): stream `reps` passes of 16-byte reads over
 * `bytes` of the device buffer `buf` (caller-owned) on `stream`; *gbs = bytes*reps/time.
 * A buffer that fits the 126 MB L2 measures the L2 read bandwidth the gather-bound
 * SpMM is limited by; a multi-GB buffer measures HBM read bandwidth. Synchronises. */
int cdfgnn_bandwidth_probe(const void* buf, int64_t bytes, int32_t reps, double* gbs, void* stream);

const char* cdfgnn_last_error(void);
const char* cdfgnn_version(void);

#ifdef __cplusplus
}
#endif
#endif /* CDFGNN_H */
