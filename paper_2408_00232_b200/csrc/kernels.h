// Device-side structures and kernel launchers of libcdfgnn (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#include "cdfgnn.h"

namespace cdfgnn {

constexpr int kMaxParts = CDFGNN_MAX_PARTS;

inline int64_t ld_of(int64_t F) { return (F + 3) / 4 * 4; }   // reading R24
inline int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }
// Bytes of one message row (kernels_halo.cu): B = 0 fp32 payload (4 ld), B = 8 one byte per
// code (ld), B = 4 two codes per byte (roundup(ld/2, 4)), B = 16 uint16 codes (2 ld).  Always a
// multiple of 4; columns F..ld-1 carry zero codes.
inline int64_t code_row_bytes(int bits, int64_t ld) {
    return bits == 0 ? 4 * ld : (bits == 8 ? ld : (bits == 4 ? align_up(ld / 2, 4) : 2 * ld));
}
// Slot-addressed message layout: 16-byte header {u32 stamp, f32 lo, f32 hi, 0} + the row.
inline int64_t slot_stride(int bits, int64_t ld) { return align_up(16 + code_row_bytes(bits, ld), 16); }

// Message regions of one part, one per peer part.  A region of capacity C holds
//   hdr: C entries of {u32 pos, f32 lo, f32 hi} (quantised) or {u32 pos} (fp32)
//   pay: at hdr + align256(C*hdr_bytes): C rows of F codes (uint8) or ld floats.
struct RegionTab {
    uint8_t* hdr[kMaxParts];
    uint8_t* pay[kMaxParts];
    int32_t* cnt[kMaxParts];   // message count slot of the region (written by the sender)
};

// Everything the halo kernels need about one local part (device pointers).
struct HaloDev {
    int32_t me, p;
    int64_t n, B, M;
    int quant;                 // bits per code: 0 (fp32 payloads), 4, 8 or 16
    int64_t hdr_bytes;         // 12 (quantised) or 4
    const int64_t* moff;       // [p+1] mirror slab offsets (mirror index space)
    const int64_t* hoff;       // [p+1] halo list offsets (master side)
    const int32_t* halo_local; // [hoff[p]] local master rows
    const RegionTab* gsend;    // mirror-role send regions (gather), per master peer
    const RegionTab* grecv;    // gather messages received, per source part
    const RegionTab* ssend;    // master-role send regions (scatter), per mirror peer
    const RegionTab* srecv;    // scatter messages received, per master part
    int remote;                // send regions live in peer GPUs' memory (NVLink push)
    uint8_t* gflag;            // [M]
    uint8_t* fired;            // [B]
    uint8_t* active;           // [B]
    int32_t* idxmap;           // [p*B]
    int32_t* mmap;             // [M]
    uint8_t* stage_codes;      // [B*Fmax] quantised scatter codes
    float* stage_lohi;         // [B*2]
    float* stage_a;            // [B*ldmax] aggregate for the no-cache fp32 scatter
    int32_t* err;              // protocol error flag (device)
    const int32_t* hpos;       // [B*p] slot layout: position of master row r in the halo list
                               // shared with part s (hpos[r*p + s]; -1: no replica on s)
};

// Slot-addressed message regions (kernels_halo.cu): base[s] = the region of the (this part,
// peer s) pair in the current phase's direction; slot k at base + k * stride holds the
// message of the vertex at halo-list position k.  nullptr for s == me.
struct SlotTab {
    uint8_t* base[kMaxParts];
};

// NVLink put: copy each peer's compacted messages (count from device memory) from local
// staging into the peer GPU's receive region through a CUDA-IPC mapping.
struct PutTab {
    const uint8_t* src_hdr[kMaxParts];
    const uint8_t* src_pay[kMaxParts];
    const int32_t* src_cnt[kMaxParts];
    uint8_t* dst_hdr[kMaxParts];      // nullptr: no peer
    uint8_t* dst_pay[kMaxParts];
    int32_t* dst_cnt[kMaxParts];
};
int launch_put(const PutTab* tab, int p, int64_t hdr_bytes, int64_t row_bytes, int64_t max_count,
               cudaStream_t s);

// Device-side barrier of the NVLink push transport: rank `me` publishes `seq` into every
// peer's arrival slot for `me` (system-scope release, through the CUDA-IPC mapping) and waits
// until each peer has published `seq` into its own slot array (system-scope acquire).  Every
// rank runs the same sequence of barriers, so `seq` is a per-context counter.  A wait longer
// than ~10 s sets *err = 5 instead of hanging.
struct BarTab {
    uint64_t* peer_slot[kMaxParts];   // peer r's arrival slot for me (mapped), nullptr for r == me
    const uint64_t* my_slots;         // [p] local arrival slots, written by the peers
    int p, me;
};
int launch_nvl_barrier(const BarTab& t, uint64_t seq, int32_t* err, cudaStream_t s);

// Cache tables of one (layer, direction) of one part (may be null with cache off).
struct CacheDev {
    float* s_mir;   // [M*ld]
    float* b_mir;   // [M*ld]
    float* s_mas;   // [B*ld]
    float* a;       // [B*ld]
    float* b_mas;   // [B*ld]
};

struct SyncArgs {
    float* X;             // part's rows [n*ld]
    int64_t ld;
    int F;
    float eps;
    int nocache;          // reading R14
    int no_msgs;          // gather phase elided (§8 f2): masters see no received messages
    int no_scatter;       // scatter phase elided (§8 f2): masters store no scatter messages
    int64_t rowb;         // code_row_bytes(quant, ld)
    int64_t stride;       // slot layout: slot_stride(quant, ld)
    uint32_t gstamp, sstamp;   // slot layout: stamps of this sync's gather / scatter messages
    int relu;             // slot layout: the synced Z rows are written as σ(Z) = max(Z, 0) (R3, fused)
    CacheDev c;
    unsigned long long* stats;  // [4]: gather_sent, master_fired, active, scatter_msgs
};

// ---- halo kernels (kernels_halo.cu)
// tiles of the gather / scatter pack launches (host-side offsets)
int gather_tiles_host(const int64_t* moff, int p, int64_t ld);
int scatter_tiles_host(const int64_t* hoff, int p);
// Each launcher returns the number of kernels it launched.
int launch_gather_pack_n(const HaloDev& h, const SyncArgs& a, int ntiles, cudaStream_t s);
// rt: the receive-side region table (host copy, passed by value as a kernel parameter so the
// message pointers need no dependent global load)
int launch_map(const HaloDev& h, const RegionTab& rt, int mirror_side, int64_t max_count, cudaStream_t s);
int launch_master(const HaloDev& h, const SyncArgs& a, const RegionTab& rt, cudaStream_t s);
int launch_scatter_pack_n(const HaloDev& h, const SyncArgs& a, int ntiles, cudaStream_t s);
int launch_mirror_apply(const HaloDev& h, const SyncArgs& a, const RegionTab& rt, cudaStream_t s);
// slot layout: gather stores each sender's message into dst.base[master part] slot pos; the
// master kernel applies src (gather) slots, its own Δ, and stores the scatter messages into
// sdst.base[mirror part]; the mirror kernel applies src (scatter) slots
int launch_gather_slot(const HaloDev& h, const SyncArgs& a, const SlotTab& dst, cudaStream_t s);
int launch_master_slot(const HaloDev& h, const SyncArgs& a, const SlotTab& src, const SlotTab& sdst,
                       cudaStream_t s);
int launch_mirror_slot(const HaloDev& h, const SyncArgs& a, const SlotTab& src, cudaStream_t s);

// ---- SpMM (kernels_spmm.cu): Y[n x ld] = Â T
// Work items in visiting order: {row, seg} (seg = -1: the whole row; else segment seg of a
// split row, CSR range [seg_beg[z + seg], seg_beg[z + seg + 1]) with split[row] = {x: first
// partial slot, y: segments, z: first seg_beg entry}; the row's last finisher sums the
// partials in segment order).  items == nullptr: identity order, no splitting.
struct SpmmItems {
    const int2* items;          // [n_items]
    const int4* split;          // [n]
    const int32_t* seg_beg;     // [segments + split rows]
    float* partial;             // [slots x width] segment partials
    int32_t* counter;           // [slots] segments finished per split row (at its first slot; zero at rest)
};
int spmm_chunk(bool wide, int64_t nnz);
int spmm_default_phases();
int spmm_phase_min_degree();
// SpMM epilogue fused with the gather of the following synchronisation (§8 f1): a row group that
// finished a mirror row [B, B+M) runs Alg. 2 L3-L9 on it from registers (test, quantise, slot
// store, snapshot, flag) — the separate gather kernel's re-read of Z disappears.
struct GatherFuse {
    HaloDev h;
    SyncArgs a;
    SlotTab dst;
};
// width (<= 1024, % 4 == 0; default ld): the columns computed; ld: row stride of T and Y.  Split-row
// partials are width floats per slot.  gf (optional): fuse the gather into the epilogue.
// relu_row0: rows >= relu_row0 (the interior rows) are written as max(Z, 0) — σ fused (R3); the
// boundary rows keep their raw partials for the synchronisation
void launch_spmm(const int32_t* rowptr, const int32_t* colidx, const float* val, int64_t n_items,
                 const SpmmItems& it, const float* T, float* Y, int64_t ld, cudaStream_t s, int64_t width = 0,
                 const GatherFuse* gf = nullptr, int64_t relu_row0 = INT64_MAX);
// stats[0] += number of set flags (uint8) among n (the fused gather's sent count)
void launch_count_flags(const uint8_t* f, int64_t n, unsigned long long* out, cudaStream_t s);

// ---- dense (kernels_dense.cu)
// C[M x ldc] = op(A) op(B) (+ mask) ; columns [N, ldc) of C are written as zero.
//   TA: A element (m,k) = A[k*lda + m], else A[m*lda + k]
//   TB: B element (k,n) = B[n*ldb + k], else B[k*ldb + n]
//   mask (optional): C(m,n) *= (mask[m*ldm + n] > 0)
void launch_gemm_simt(bool TA, bool TB, int64_t M, int64_t N, int64_t K, const float* A,
                      int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc,
                      const float* mask, int64_t ldm, float* splitk_ws, int64_t splitk_cap,
                      bool accumulate, cudaStream_t s);
// tcgen05 TF32 GEMMs (gemm_tc.cu); return a CDFGNN status
int launch_pad_rows(const float* src, int64_t rows, int64_t cols, float* dst, int64_t ldd, cudaStream_t s);
int launch_relu_transpose(const float* Z, int64_t rows, int64_t cols, int64_t ldz, float* H, float* Ht,
                          int64_t ldt, cudaStream_t s);
int launch_transpose(const float* src, int64_t rows, int64_t cols, int64_t lds, float* dst, int64_t ldd,
                     cudaStream_t s);
// split3: 3xTF32 (A_hi·B_hi + A_hi·B_lo + A_lo·B_hi, ~fp32 accuracy); else 1xTF32 (RN inputs)
int gemm_tc_fwd(int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, const float* Bt, int64_t ldb,
                float* C, int64_t ldc, bool split3, cudaStream_t s);
int gemm_tc_bwd_data(int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, const float* Bk, int64_t ldb,
                     float* C, int64_t ldc, const float* mask, int64_t ldm, bool split3, cudaStream_t s);
int gemm_tc_wgrad(int64_t M, int64_t N, int64_t K, const float* Ht, int64_t ldh, const float* St, int64_t lds,
                  float* C, int64_t ldc, float* ws, int64_t ws_cap, bool accumulate, bool split3,
                  cudaStream_t s, int* launches);
// out[k] = X[idx[k]] rows (ld floats, ld % 4 == 0), k < count; returns the launch count
int launch_gather_rows(const float* X, int64_t ld, const int32_t* idx, int64_t count, float* out, cudaStream_t s);
int gemm_tc_wgrad_mn(int64_t M, int64_t N, int64_t K, const float* H, int64_t ldh, const float* S, int64_t lds,
                     float* C, int64_t ldc, float* ws, int64_t ws_cap, bool accumulate, bool split3,
                     cudaStream_t s, int* launches);
void launch_read_probe(const float4* p, int64_t n4, int reps, float* sink, cudaStream_t s);
void launch_relu(const float* Z, float* H, int64_t count, cudaStream_t s);
void launch_loss(const float* logits, int64_t ld, int C, int64_t n, int64_t B, int64_t M,
                 const int32_t* labels, const uint8_t* train, double inv_ntrain, float* dlogits,
                 float* rowloss, int* correct, int* err, cudaStream_t s);
// out = Σ rowloss[0..n) in fp64, fixed order (part: scratch of 148 doubles); two launches
void launch_reduce_rows(const float* rowloss, int64_t n, double* out, double* part, cudaStream_t s);
void launch_count_train(int64_t n, int64_t B, int64_t M, const uint8_t* train, int* out,
                        cudaStream_t s);
// err (device, may be NULL): the update is skipped when *err != 0 (protocol / data error)
void launch_optimizer(int kind, float* W, const float* G, float* m, float* v, int64_t count,
                      float lr, float b1, float b2, float eps, float bc1, float bc2,
                      const int32_t* err, cudaStream_t s);

}  // namespace cdfgnn
