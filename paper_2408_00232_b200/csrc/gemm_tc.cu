// tcgen05 TF32 tensor-core GEMMs for the dense feature transform and its gradients.
//
//   T  = H W                  (eq. 1; R5 Â(HW))        A = H,  B = Wᵀ (padded copy)
//   δ̈  = (S Wᵀ) ⊙ 𝟙[H > 0]    (R3, R6)              A = S,  B = W  (padded copy)
//   ∇W = Hᵀ S                 (eq. 5; R6), split-K  A = H, B = S read in place (MN-major);
//                                                              K-major transposed copies only with
//                                                              CDFGNN_WGRAD_KMAJOR=1
// T = HW and δ̈ feed K-major operands; ∇W reads H and S in place as MN-major operands, which
// for tf32 the UMMA accepts only in the 128-B swizzle with 32-B atoms (layout type 1, 4 k-rows
// per atom) — with the plain 128-B swizzle the accumulators came back zero.
//
// One CTA computes a 128 x BN fp32 tile over a K range: warp 0 issues TMA loads
// (64-byte swizzled K-major boxes of 16 k, 128-byte / 32-B-atom MN-major boxes) into a
// STAGES-deep shared-memory ring guarded by mbarriers; warps 2-5 split each fp32 stage into
// tf32 hi (the raw word) + lo (3xTF32); one elected thread of warp 1 issues
// tcgen05.mma.kind::tf32 (M = 128, N = BN, K = 8) into a double-buffered TMEM accumulator,
// tcgen05.commit releasing ring slots; warps 6-13 read the accumulator with tcgen05.ld and run
// the epilogue (mask, zero padding columns, split-K partials, TMA stores).  3xTF32 GEMMs run
// on CTA pairs (PAIR: cluster of 2, cta_group::2, M = 256): each CTA loads and converts its
// 128 rows of A and half of B, the leader issues the MMAs over both CTAs' shared memory, which
// halves each SM's shared-memory operand and conversion traffic for B — the single-CTA
// kernel's limit.  Split-K partials are summed in a fixed order by a separate kernel, so
// results are run-to-run deterministic.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>

#include "common.h"
#include "kernels.h"

namespace cdfgnn {
namespace {

constexpr int BM = 128;
#ifndef GEMM_BK
#define GEMM_BK 16
#endif
// k-block: 16 tf32 = 64-byte K-major rows (64-B swizzle), so a 3xTF32 stage at N = 256 is 48 KB
// and four stages fit where two 32-wide ones did (32 = 128-byte rows, 128-B swizzle)
constexpr int BK = GEMM_BK;
static_assert(BK == 16 || BK == 32, "BK is 16 or 32");
constexpr uint32_t kKLayout = BK == 32 ? 2u : 4u;     // UMMA layout type: SWIZZLE_128B / SWIZZLE_64B
constexpr uint32_t kKSbo = 8 * BK * 4;                 // K-major: bytes between 8-row core-matrix groups
constexpr int kConvWarps = 4;     // 3xTF32 converter warps
constexpr int kEpiWarps = 8;      // two epilogue warpgroups split each tile's column chunks
constexpr int kEpiWarp0 = 2 + kConvWarps;
constexpr int kThreads = 32 * (2 + kConvWarps + kEpiWarps);   // TMA, MMA, converters, epilogue
#ifndef GEMM_MN_LBO
#define GEMM_MN_LBO (BK * 128)   // MN-major: byte stride between 32-element MN chunks
#endif
#ifndef GEMM_MN_SBO
#define GEMM_MN_SBO 512          // MN-major: byte stride between groups of 4 k-rows (32-B-atom swizzle)
#endif

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}

// TMA bulk store of a 32 x 32 fp32 box from 128-B-swizzled shared memory
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(smem_u32(src)), "r"(c0), "r"(c1)
                 : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// arrive on the mbarrier at the same shared-memory offset in CTA `rank` of the cluster
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* bar, uint32_t rank) {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(rank));
    // default (.release.cta) semantics as CUTLASS's ClusterBarrier::arrive: .release.cluster
    // compiles to MEMBAR.GPU + ERRBAR per arrive and halved the pair GEMM's throughput
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAITC_%=:\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAITC_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// MMA completion -> the mbarrier at this offset in both CTAs of the pair
__device__ __forceinline__ void tc_commit_pair(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                     smem_u32(bar)),
                 "h"((uint16_t)3)
                 : "memory");
}
__device__ __forceinline__ void tc_mma_tf32_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                 uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tc_mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// 128-byte-swizzled shared-memory matrix descriptor (sm_100 UMMA, version 1)
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout = 2) {
    uint64_t d = 0;
    d |= (uint64_t)((addr & 0x3FFFFu) >> 4);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;          // descriptor version (sm_100)
    d |= (uint64_t)layout << 61;     // 2 = SWIZZLE_128B (K-major); 1 = SWIZZLE_128B_BASE32B (MN-major tf32)
    return d;
}
// MN-major tf32 operands: the only smem layout the UMMA accepts is 128-B swizzle with 32-B atoms
// (CUTLASS sm100_common.inl), 4 k-rows per swizzle atom: SBO = 512 B, LBO = 4 KB between the
// 32-wide MN chunks of a stage, +1024 B per 8 k-rows
__device__ __forceinline__ uint64_t smem_desc_mn(uint32_t addr) { return smem_desc(addr, GEMM_MN_LBO, GEMM_MN_SBO, 1); }

// 32 lanes x 32 consecutive 32-bit TMEM columns -> 32 registers per thread
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
          "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
          "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

template <int BN, bool SPLIT3, bool PAIR = false>
struct Cfg {
    static constexpr int BNL = PAIR ? BN / 2 : BN;                      // B rows held by this CTA
    static constexpr int A_BYTES = BM * BK * 4;
    static constexpr int B_BYTES = BNL * BK * 4;
    static constexpr int TMA_BYTES = A_BYTES + B_BYTES;                  // fp32 (or tf32) tiles
    static constexpr int STAGE_BYTES = TMA_BYTES * (SPLIT3 ? 2 : 1);     // + lo parts for 3xTF32
    static constexpr int STAGES_FIT = (SPLIT3 ? 196608 : 200704) / STAGE_BYTES;
    static constexpr int STAGES = STAGES_FIT > 8 ? 8 : STAGES_FIT;   // 3 mbarriers per stage in 256 B
    static constexpr int EPI_BYTES = kEpiWarps * 32 * 32 * 4;            // epilogue staging (TMA store boxes)
    static constexpr int SMEM = STAGES * STAGE_BYTES + EPI_BYTES + 1024 /*align*/ + 256 /*barriers*/;
    static constexpr int TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;        // double-buffered accumulator
};

#ifndef GEMM_PAIR_DEFAULT
#define GEMM_PAIR_DEFAULT 1
#endif
// CTA-pair 3xTF32 GEMMs (CDFGNN_GEMM_PAIR=0/1 overrides GEMM_PAIR_DEFAULT)
bool gemm_pair_on() {
    static const bool v = [] { const char* e = getenv("CDFGNN_GEMM_PAIR"); return e ? atoi(e) != 0 : GEMM_PAIR_DEFAULT != 0; }();
    return v;
}
#ifndef GEMM_HI_INPLACE
#define GEMM_HI_INPLACE 0
#endif
__device__ __forceinline__ float tf32_tr(float x) { return __uint_as_float(__float_as_uint(x) & ~0x1FFFu); }
__device__ __forceinline__ float tf32_rn(float x) {
    uint32_t u = __float_as_uint(x);
    u = (u + 0xFFFu + ((u >> 13) & 1u)) & ~0x1FFFu;      // round to nearest even, 10-bit mantissa
    return __uint_as_float(u);
}

struct EpiArgs {
    float* C;          // output (or nullptr with ws)
    int64_t ldc;
    const float* mask; // optional: C *= (mask > 0)
    int64_t ldm;
    float* ws;         // split-K partials [z][M][ldw]
    int64_t ldw;
    int accumulate;
    int tma;           // 1: stores through the C tensor map (2-D {ldc, M}; 3-D {ldw, M, splits} for ws)
};

// Persistent, warp-specialised tcgen05 GEMM.  One CTA per SM walks the output tiles
// (m fastest-changing over n so neighbouring CTAs share A tiles in L2):
//   warp 0          TMA producer (STAGES-deep smem ring, mbarrier full/empty)
//   warp 1          MMA issuer (one elected thread), accumulator double-buffered in TMEM
//                   (2 x BN columns) so the epilogue of tile i overlaps the MMAs of tile i+1
//   warps 2-5       3xTF32 converters: fp32 tile -> tf32 hi (in place) + lo (second buffer)
//   warps 6-9       epilogue: tcgen05.ld 32 lanes each -> mask / zero padding / split-K partial
// PAIR: a CTA pair (cluster of 2, cta_group::2) computes a 256 x BN tile — each CTA loads and
// converts its 128 rows of A and half of B's BN rows, the leader issues M = 256 MMAs that read
// both CTAs' shared memory, and each CTA's TMEM holds its 128 accumulator rows.  Per SM this
// halves the B-operand reads and the converter traffic for B.
template <bool A_MN, bool B_MN, int BN, bool SPLIT3, bool PAIR>
__global__ void __launch_bounds__(kThreads, 1)
gemm_tf32_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 const __grid_constant__ CUtensorMap tmC, int M, int N, int total_kb, int kb_per_split, int m_tiles,
                 int n_tiles, int z_tiles, EpiArgs ep) {
    using C_ = Cfg<BN, SPLIT3, PAIR>;
    static_assert(!PAIR || SPLIT3, "the CTA pair is built for the 3xTF32 path");
    constexpr int BMT = PAIR ? 2 * BM : BM;                 // output tile rows
    constexpr int NCTA = PAIR ? 2 : 1;
    const uint32_t crank = PAIR ? cluster_ctarank() : 0u;
    const bool leader = crank == 0;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    // stage s: [A (hi)][B (hi)][A lo][B lo]   (lo parts only with SPLIT3)
    auto stA = [&](int st) { return smem + st * C_::STAGE_BYTES; };
    auto stB = [&](int st) { return smem + st * C_::STAGE_BYTES + C_::A_BYTES; };
    float* epi_smem = reinterpret_cast<float*>(smem + C_::STAGES * C_::STAGE_BYTES);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + C_::STAGES * C_::STAGE_BYTES + C_::EPI_BYTES);
    uint64_t* empty = full + C_::STAGES;
    uint64_t* conv = empty + C_::STAGES;
    uint64_t* tfull = conv + C_::STAGES;      // [2] accumulator ready
    uint64_t* tempty = tfull + 2;             // [2] accumulator drained
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int total_tiles = m_tiles * n_tiles * z_tiles;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < C_::STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
            mbar_init(&conv[s], kConvWarps * NCTA);   // one arrival per converter warp (both CTAs)
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], kEpiWarps * NCTA);   // one arrival per epilogue warp (both CTAs)
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    }
    if (warp == 1) {
        if (PAIR) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                         "n"(C_::TMEM_COLS)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                         "n"(C_::TMEM_COLS)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
    }
    tc_fence_before();
    __syncthreads();
    if (PAIR) cluster_sync_all();             // the peer's barriers exist before any remote arrive
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    auto decode = [&](int t, int& m0, int& n0, int& kb0, int& nkb) {
        const int mn = m_tiles * n_tiles;
        const int z = t / mn;
        const int r = t - z * mn;
        const int nt = r / m_tiles;
        const int mt = r - nt * m_tiles;
        m0 = mt * BMT;
        n0 = nt * BN;
        kb0 = z * kb_per_split;
        nkb = min(total_kb, kb0 + kb_per_split) - kb0;
    };

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer ----------------
            int it = 0;
            for (int t = blockIdx.x / NCTA; t < total_tiles; t += gridDim.x / NCTA) {
                int m0, n0, kb0, nkb;
                decode(t, m0, n0, kb0, nkb);
                for (int i = 0; i < nkb; ++i, ++it) {
                    const int s = it % C_::STAGES;
                    const uint32_t ph = (uint32_t)(it / C_::STAGES) & 1u;
                    mbar_wait(&empty[s], ph ^ 1u);
                    mbar_expect_tx(&full[s], C_::TMA_BYTES);
                    const int k = (kb0 + i) * BK;
                    uint8_t* a = stA(s);
                    uint8_t* b = stB(s);
                    const int ma = m0 + BM * (int)crank;             // this CTA's 128 rows of A
                    const int nb = n0 + C_::BNL * (int)crank;        // and its BNL rows of B
                    if (!A_MN) {
                        tma_load_2d(a, &tmA, &full[s], k, ma);                      // box {BK k, 128 m}
                    } else {
#pragma unroll
                        for (int c = 0; c < BM / 32; ++c)
                            tma_load_2d(a + c * BK * 128, &tmA, &full[s], ma + 32 * c, k);
                    }
                    if (!B_MN) {
                        tma_load_2d(b, &tmB, &full[s], k, nb);                      // box {BK k, BNL n}
                    } else {
#pragma unroll
                        for (int c = 0; c < C_::BNL / 32; ++c)
                            tma_load_2d(b + c * BK * 128, &tmB, &full[s], nb + 32 * c, k);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && leader) {
            // ---------------- MMA issuer (the pair's leader) ----------------
            constexpr uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((A_MN ? 1u : 0u) << 15) |
                                       ((B_MN ? 1u : 0u) << 16) | ((uint32_t)(BN >> 3) << 17) |
                                       ((uint32_t)(BMT >> 4) << 24);
            int it = 0, ti = 0;
            for (int t = blockIdx.x / NCTA; t < total_tiles; t += gridDim.x / NCTA, ++ti) {
                int m0, n0, kb0, nkb;
                decode(t, m0, n0, kb0, nkb);
                const int acc = ti & 1;
                const uint32_t aph = (uint32_t)(ti >> 1) & 1u;
                if (PAIR) mbar_wait_cluster(&tempty[acc], aph ^ 1u);   // both CTAs' epilogues drained it
                else mbar_wait(&tempty[acc], aph ^ 1u);         // epilogue drained this accumulator
                tc_fence_after();
                const uint32_t dcol = tmem + (uint32_t)(acc * BN);
                for (int i = 0; i < nkb; ++i, ++it) {
                    const int s = it % C_::STAGES;
                    const uint32_t ph = (uint32_t)(it / C_::STAGES) & 1u;
                    if (PAIR) mbar_wait_cluster(&conv[s], ph);       // both CTAs' stages converted
                    else mbar_wait(SPLIT3 ? &conv[s] : &full[s], ph);
                    tc_fence_after();
                    const uint32_t a_base = smem_u32(stA(s));
                    const uint32_t b_base = smem_u32(stB(s));
                    if (SPLIT3) {
                        // 3xTF32: A_hi·B_hi + A_hi·B_lo + A_lo·B_hi
                        const uint32_t alo = a_base + C_::TMA_BYTES, blo = b_base + C_::TMA_BYTES;
#pragma unroll
                        for (int kk = 0; kk < BK / 8; ++kk) {
                            const uint64_t ah = A_MN ? smem_desc_mn(a_base + kk * 1024) : smem_desc(a_base + kk * 32, 16, kKSbo, kKLayout);
                            const uint64_t bh = B_MN ? smem_desc_mn(b_base + kk * 1024) : smem_desc(b_base + kk * 32, 16, kKSbo, kKLayout);
                            const uint64_t al = A_MN ? smem_desc_mn(alo + kk * 1024) : smem_desc(alo + kk * 32, 16, kKSbo, kKLayout);
                            const uint64_t bl = B_MN ? smem_desc_mn(blo + kk * 1024) : smem_desc(blo + kk * 32, 16, kKSbo, kKLayout);
                            if (PAIR) {
                                tc_mma_tf32_pair(dcol, ah, bh, idesc, (i > 0 || kk > 0) ? 1u : 0u);
                                tc_mma_tf32_pair(dcol, ah, bl, idesc, 1u);
                                tc_mma_tf32_pair(dcol, al, bh, idesc, 1u);
                            } else {
                                tc_mma_tf32(dcol, ah, bh, idesc, (i > 0 || kk > 0) ? 1u : 0u);
                                tc_mma_tf32(dcol, ah, bl, idesc, 1u);
                                tc_mma_tf32(dcol, al, bh, idesc, 1u);
                            }
                        }
                    } else {
#pragma unroll
                        for (int kk = 0; kk < BK / 8; ++kk) {
                            // K-major: +32 B per 8 tf32 inside the 64-/128-B swizzle row (SBO = 8 rows)
                            // MN-major: +1024 B per 8 k-rows (LBO = stride of 32-wide MN chunks)
                            const uint64_t ad = A_MN ? smem_desc_mn(a_base + kk * 1024)
                                                     : smem_desc(a_base + kk * 32, 16, kKSbo, kKLayout);
                            const uint64_t bd = B_MN ? smem_desc_mn(b_base + kk * 1024)
                                                     : smem_desc(b_base + kk * 32, 16, kKSbo, kKLayout);
                            tc_mma_tf32(dcol, ad, bd, idesc, (i > 0 || kk > 0) ? 1u : 0u);
                        }
                    }
                    if (PAIR) tc_commit_pair(&empty[s]);   // both CTAs' slots free once read
                    else tc_commit(&empty[s]);       // slot free once these MMAs have read it
                }
                if (PAIR) tc_commit_pair(&tfull[acc]);
                else tc_commit(&tfull[acc]);    // accumulator complete
            }
        }
    } else if (warp < kEpiWarp0) {
        if (SPLIT3) {
            // ---------------- converters: fp32 -> tf32 hi (in place) + lo ----------------
            const int ct = threadIdx.x - 64;                 // 0 .. 32*kConvWarps-1
            constexpr int NV = C_::TMA_BYTES / 16;           // float4 per stage (A and B)
            int it = 0;
            for (int t = blockIdx.x / NCTA; t < total_tiles; t += gridDim.x / NCTA) {
                int m0, n0, kb0, nkb;
                decode(t, m0, n0, kb0, nkb);
                for (int i = 0; i < nkb; ++i, ++it) {
                    const int s = it % C_::STAGES;
                    const uint32_t ph = (uint32_t)(it / C_::STAGES) & 1u;
                    mbar_wait(&full[s], ph);
                    float4* base = reinterpret_cast<float4*>(stA(s));
                    float4* lo = reinterpret_cast<float4*>(stA(s) + C_::TMA_BYTES);
                    const uint32_t hi_s = smem_u32(stA(s)), lo_s = hi_s + (uint32_t)C_::TMA_BYTES;
                    (void)hi_s; (void)lo_s; (void)base; (void)lo;
#pragma unroll 4
                    for (int v = ct; v < NV; v += 32 * kConvWarps) {
#if GEMM_HI_INPLACE
                        const float4 x = base[v];
                        float4 h, l;
                        h.x = tf32_rn(x.x); h.y = tf32_rn(x.y); h.z = tf32_rn(x.z); h.w = tf32_rn(x.w);
                        l.x = x.x - h.x; l.y = x.y - h.y; l.z = x.z - h.z; l.w = x.w - h.w;
                        base[v] = h;
                        lo[v] = l;
#else
                        // hi = the raw fp32 word: kind::tf32 reads only its top 19 bits (truncation,
                        // experiments/tc_raw.cu), so lo = x − trunc(x) is exact and only lo is written.
                        // Explicit shared-window ld/st: the generic LD/ST forms cost 1-3 % of the GEMM
                        // phase (profiles/r2/experiments/gemm_converter_ab.txt)
                        float4 x, l;
                        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                                     : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w) : "r"(hi_s + 16u * v));
                        l.x = x.x - tf32_tr(x.x); l.y = x.y - tf32_tr(x.y);
                        l.z = x.z - tf32_tr(x.z); l.w = x.w - tf32_tr(x.w);
                        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(lo_s + 16u * v), "f"(l.x), "f"(l.y),
                                     "f"(l.z), "f"(l.w)
                                     : "memory");
#endif
                    }
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // visible to tcgen05
                    __syncwarp();
                    if (lane == 0) {
                        if (PAIR) mbar_arrive_remote(&conv[s], 0);   // the leader's barrier (own CTA too)
                        else asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&conv[s])) : "memory");
                    }
                }
            }
        }
    } else {
        // ---------------- epilogue warps ----------------
        const int q = warp & 3;             // TMEM lane quarter this warp may access
        const int eg = (warp - kEpiWarp0) >> 2;   // epilogue warpgroup: even / odd 32-column chunks
        int ti = 0;
        for (int t = blockIdx.x / NCTA; t < total_tiles; t += gridDim.x / NCTA, ++ti) {
            int m0, n0, kb0, nkb;
            decode(t, m0, n0, kb0, nkb);
            const int acc = ti & 1;
            const uint32_t aph = (uint32_t)(ti >> 1) & 1u;
            mbar_wait(&tfull[acc], aph);
            tc_fence_after();
            // each lane holds one accumulator row (32 consecutive columns per tcgen05.ld)
            float* st = epi_smem + (warp - kEpiWarp0) * 32 * 32;     // 4 KB, 1024-B aligned
            const int rbase = m0 + BM * (int)crank + 32 * q;
            const int row = rbase + lane;
            const int64_t ldo = ep.ws ? ep.ldw : ep.ldc;
            const int z = t / (m_tiles * n_tiles);
#pragma unroll 1
            for (int c0 = 32 * eg; c0 < BN; c0 += 64) {
                const int col0 = n0 + c0;
                if (col0 >= ldo) break;                        // warp-uniform
                // masks for this lane's row segment, in flight with the TMEM load
                float4 mk[8];
                if (ep.mask) {
                    const float* mrow = ep.mask + (int64_t)row * ep.ldm + col0;
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        mk[j] = (row < M && col0 + 4 * j < ldo) ? *reinterpret_cast<const float4*>(mrow + 4 * j)
                                                               : make_float4(1.f, 1.f, 1.f, 1.f);
                }
                float v[32];
                tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(acc * BN + c0), v);
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    if (col0 + j >= N) v[j] = 0.f;             // zero padding columns
                    if (ep.mask) {
                        const float mj = (j & 3) == 0 ? mk[j >> 2].x : (j & 3) == 1 ? mk[j >> 2].y
                                       : (j & 3) == 2 ? mk[j >> 2].z : mk[j >> 2].w;
                        if (!(mj > 0.f)) v[j] = 0.f;
                    }
                }
                if (ep.tma) {
                    // 128-B swizzled 32 x 32 box: lane r's 16-byte chunk j lives at chunk j ^ (r & 7)
                    if (lane == 0) bulk_wait_read0();           // the previous box has left st
                    __syncwarp();
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        *reinterpret_cast<float4*>(st + lane * 32 + ((j ^ (lane & 7)) * 4)) =
                            make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) {
                        if (ep.ws) tma_store_3d(&tmC, st, col0, rbase, z);
                        else tma_store_2d(&tmC, st, col0, rbase);
                        bulk_commit();
                    }
                } else if (row < M) {
                    float* obase = ep.ws ? ep.ws + (int64_t)z * M * ep.ldw : ep.C;
                    float* orow = obase + (int64_t)row * ldo;
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const int col = col0 + j;
                        if (col >= ldo) break;
                        float o = v[j];
                        if (ep.accumulate && !ep.ws && col < N) o += orow[col];
                        orow[col] = o;
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (PAIR) mbar_arrive_remote(&tempty[acc], 0);
                else asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tempty[acc])) : "memory");
            }
        }
    }
    if (warp >= kEpiWarp0 && lane == 0) bulk_wait0();      // TMA stores complete before exit
    tc_fence_before();
    __syncthreads();
    if (PAIR) cluster_sync_all();     // the leader's MMAs have read this CTA's shared memory
    if (warp == 1) {
        tc_fence_after();
        if (PAIR)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C_::TMEM_COLS)
                         : "memory");
        else
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C_::TMEM_COLS)
                         : "memory");
    }
}

// one warp per output element: lane j sums partials j, j+32, ... then a fixed xor tree — a fixed
// order (run-to-run deterministic) without a 100+-long dependent load chain per element
__global__ void splitk_sum_warp_kernel(int64_t M, int64_t N, int64_t ldw, int splits, const float* __restrict__ ws,
                                       float* __restrict__ C, int64_t ldc, int accumulate) {
    const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= M * ldc) return;
    const int64_t m = i / ldc, n = i % ldc;
    if (n >= N) {
        if (lane == 0) C[i] = 0.f;
        return;
    }
    float v = 0.f;
    for (int z = lane; z < splits; z += 32) v += ws[((int64_t)z * M + m) * ldw + n];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) C[i] = accumulate ? v + C[i] : v;
}

__global__ void splitk_sum_kernel(int64_t M, int64_t N, int64_t ldw, int splits, const float* __restrict__ ws,
                                  float* __restrict__ C, int64_t ldc, int accumulate) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= M * ldc) return;
    const int64_t m = i / ldc, n = i % ldc;
    if (n >= N) { C[i] = 0.f; return; }
    float v = 0.f;
    for (int z = 0; z < splits; ++z) v += ws[((int64_t)z * M + m) * ldw + n];   // fixed order
    if (accumulate) v += C[i];
    C[i] = v;
}

// dst[c][r] = src[r][c]  (r < rows, c < cols), 32 x 32 tiles through shared memory
__global__ void transpose_kernel(const float* __restrict__ src, int64_t rows, int64_t cols, int64_t lds,
                                 float* __restrict__ dst, int64_t ldd) {
    __shared__ float tile[32][33];
    const int64_t r0 = (int64_t)blockIdx.x * 32, c0 = (int64_t)blockIdx.y * 32;   // rows on grid.x
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int64_t r = r0 + i, c = c0 + threadIdx.x;
        tile[i][threadIdx.x] = (r < rows && c < cols) ? src[r * lds + c] : 0.f;
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int64_t c = c0 + i, r = r0 + threadIdx.x;
        if (c < cols && r < rows) dst[c * ldd + r] = tile[threadIdx.x][i];
    }
}

// H = max(Z, 0) row-major (rows x ldz, all ldz columns) and Hᵀ [cols x ldt] in one pass
__global__ void relu_transpose_kernel(const float* __restrict__ Z, int64_t rows, int64_t cols, int64_t ldz,
                                      float* __restrict__ H, float* __restrict__ Ht, int64_t ldt) {
    __shared__ float tile[32][33];
    const int64_t r0 = (int64_t)blockIdx.x * 32, c0 = (int64_t)blockIdx.y * 32;   // rows on grid.x
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int64_t r = r0 + i, c = c0 + threadIdx.x;
        float v = 0.f;
        if (r < rows && c < ldz) {
            v = fmaxf(Z[r * ldz + c], 0.f);
            H[r * ldz + c] = v;
        }
        tile[i][threadIdx.x] = v;
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int64_t c = c0 + i, r = r0 + threadIdx.x;
        if (c < cols && r < rows) Ht[c * ldt + r] = tile[threadIdx.x][i];
    }
}

// 64 x 64 tiles, 16-byte loads and stores, 4 in flight per thread each way (the 32 x 32 scalar
// kernels above reached ~60% of HBM on the C4 wide transposes).  RELU: also writes
// H = max(Z, 0) row-major over all lds columns.  Needs lds, ldd % 4 == 0 and 16-B aligned bases.
template <bool RELU>
__global__ void __launch_bounds__(256) transpose64_kernel(const float* src, int64_t rows,   // src may alias H
                                                          int64_t cols, int64_t lds, float* H,
                                                          float* __restrict__ dst, int64_t ldd) {
    __shared__ float tile[64][65];
    const int64_t r0 = (int64_t)blockIdx.x * 64, c0 = (int64_t)blockIdx.y * 64;
    const int t = threadIdx.x;
    const int cq = t & 15, rr = t >> 4;
    float4 v[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t r = r0 + rr + 16 * i, c = c0 + 4 * cq;
        v[i] = (r < rows && c < lds) ? *reinterpret_cast<const float4*>(src + r * lds + c)
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        if (RELU) {
            v[i].x = fmaxf(v[i].x, 0.f); v[i].y = fmaxf(v[i].y, 0.f);
            v[i].z = fmaxf(v[i].z, 0.f); v[i].w = fmaxf(v[i].w, 0.f);
            const int64_t r = r0 + rr + 16 * i, c = c0 + 4 * cq;
            if (r < rows && c < lds) *reinterpret_cast<float4*>(H + r * lds + c) = v[i];
        }
        float* tr = &tile[rr + 16 * i][4 * cq];
        tr[0] = v[i].x; tr[1] = v[i].y; tr[2] = v[i].z; tr[3] = v[i].w;
    }
    __syncthreads();
    const int rq = t & 15;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int oc = (t >> 4) + 16 * j;
        const int64_t c = c0 + oc, r = r0 + 4 * rq;
        if (c >= cols || r >= rows) continue;
        const float4 o = make_float4(tile[4 * rq][oc], tile[4 * rq + 1][oc], tile[4 * rq + 2][oc], tile[4 * rq + 3][oc]);
        float* dp = dst + c * ldd + r;
        if (r + 3 < rows) {
            *reinterpret_cast<float4*>(dp) = o;
        } else {
            dp[0] = o.x;
            if (r + 1 < rows) dp[1] = o.y;
            if (r + 2 < rows) dp[2] = o.z;
        }
    }
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

__global__ void pad_rows_kernel(const float* __restrict__ src, int64_t rows, int64_t cols, float* __restrict__ dst,
                                int64_t ldd) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= rows * ldd) return;
    const int64_t r = i / ldd, c = i % ldd;
    dst[i] = c < cols ? src[r * cols + c] : 0.f;
}

// ---- host: tensor maps ----------------------------------------------------------
typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
    static EncodeFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    }
    return fn;
}

// 2-D fp32 row-major matrix [rows x cols] with row stride ld (elements); box {bc, br}
bool make_map(CUtensorMap* m, const float* base, int64_t rows, int64_t cols, int64_t ld, int bc, int br,
              bool raw_fp32 = false, bool mn_major = false) {
    EncodeFn fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)(ld * 4)};
    cuuint32_t box[2] = {(cuuint32_t)bc, (cuuint32_t)br};
    cuuint32_t es[2] = {1, 1};
    CUresult r = fn(m, raw_fp32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_TFLOAT32, 2, const_cast<float*>(base), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE,
                    mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B
                             : (BK == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B),
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// Output map for the TMA-store epilogue: fp32 [z][rows][cols] (row stride ld), box {32, 32, 1},
// 128-B swizzle; out-of-range rows / columns of a box are clipped by the TMA unit.
bool make_store_map(CUtensorMap* m, const float* base, int64_t rows, int64_t cols, int64_t ld, int64_t zs,
                    bool three_d) {
    EncodeFn fn = encode_fn();
    if (!fn || (reinterpret_cast<uintptr_t>(base) & 15) || (ld & 3)) return false;
    cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)zs};
    cuuint64_t strides[2] = {(cuuint64_t)(ld * 4), (cuuint64_t)(ld * 4 * rows)};
    cuuint32_t box[3] = {32, 32, 1};
    cuuint32_t es[3] = {1, 1, 1};
    const cuuint32_t rank = three_d ? 3 : 2;
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, const_cast<float*>(base), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

template <bool A_MN, bool B_MN, int BN, bool SPLIT3, bool PAIR = false>
int launch_variant(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc, int64_t M, int64_t N,
                   int64_t K, int splits, const EpiArgs& ep, cudaStream_t s) {
    using C_ = Cfg<BN, SPLIT3, PAIR>;
    static bool attr = false;
    auto kern = gemm_tf32_kernel<A_MN, B_MN, BN, SPLIT3, PAIR>;
    if (!attr) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C_::SMEM) != cudaSuccess)
            return CDFGNN_ECUDA;
        attr = true;
    }
    const int total_kb = (int)((K + BK - 1) / BK);
    const int kbps = (total_kb + splits - 1) / splits;
    const int zs = std::max((total_kb + kbps - 1) / kbps, 1);
    constexpr int BMT = PAIR ? 2 * BM : BM;
    const int mt = (int)((M + BMT - 1) / BMT), nt = (int)((N + BN - 1) / BN);
    const int64_t tiles = (int64_t)mt * nt * zs;
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    if (PAIR) {
        // clusters of two CTAs (one TPC), one pair per output tile at a time; the persistent grid
        // is the number of pairs that can be co-resident (not every TPC may host one), else the
        // clusters of a second wave would each redo a full share of tiles
        static int max_clusters = 0;
        cudaLaunchConfig_t lc = {};
        lc.blockDim = dim3(kThreads);
        lc.dynamicSmemBytes = C_::SMEM;
        lc.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        if (!max_clusters) {
            lc.gridDim = dim3(2 * (sms / 2));
            int mc = 0;
            if (cudaOccupancyMaxActiveClusters(&mc, kern, &lc) != cudaSuccess || mc <= 0) mc = sms / 2;
            max_clusters = std::min(mc, sms / 2);
            if (getenv("CDFGNN_GEMM_PAIR_VERBOSE")) fprintf(stderr, "gemm pair: %d co-resident clusters\n", mc);
        }
        const unsigned grid = (unsigned)(2 * std::min<int64_t>(tiles, max_clusters));
        lc.gridDim = dim3(grid);
        if (cudaLaunchKernelEx(&lc, kern, ta, tb, tc, (int)M, (int)N, total_kb, kbps, mt, nt, zs, ep) != cudaSuccess)
            return CDFGNN_ECUDA;
        return cudaGetLastError() == cudaSuccess ? CDFGNN_OK : CDFGNN_ECUDA;
    }
    const unsigned grid = (unsigned)std::min<int64_t>(tiles, sms);
    kern<<<grid, kThreads, C_::SMEM, s>>>(ta, tb, tc, (int)M, (int)N, total_kb, kbps, mt, nt, zs, ep);
    return cudaGetLastError() == cudaSuccess ? CDFGNN_OK : CDFGNN_ECUDA;
}

template <bool A_MN, bool B_MN>
int launch_bn(int BN, bool split3, const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc, int64_t M,
              int64_t N, int64_t K, int splits, const EpiArgs& ep, cudaStream_t s) {
    if (split3 && gemm_pair_on() && BN >= 128) {
        if (BN == 128) return launch_variant<A_MN, B_MN, 128, true, true>(ta, tb, tc, M, N, K, splits, ep, s);
        return launch_variant<A_MN, B_MN, 256, true, true>(ta, tb, tc, M, N, K, splits, ep, s);
    }
    if (split3) {
        if (BN == 64) return launch_variant<A_MN, B_MN, 64, true>(ta, tb, tc, M, N, K, splits, ep, s);
        if (BN == 128) return launch_variant<A_MN, B_MN, 128, true>(ta, tb, tc, M, N, K, splits, ep, s);
        return launch_variant<A_MN, B_MN, 256, true>(ta, tb, tc, M, N, K, splits, ep, s);
    }
    if (BN == 64) return launch_variant<A_MN, B_MN, 64, false>(ta, tb, tc, M, N, K, splits, ep, s);
    if (BN == 128) return launch_variant<A_MN, B_MN, 128, false>(ta, tb, tc, M, N, K, splits, ep, s);
    return launch_variant<A_MN, B_MN, 256, false>(ta, tb, tc, M, N, K, splits, ep, s);
}

// 3xTF32 at N = 256 keeps two 96 KB stages; the wider MMA halves the shared-memory
// operand traffic per flop (GEMM_SPLIT3_BN256=0 restores the 128-wide tile)
#ifndef GEMM_SPLIT3_BN256
#define GEMM_SPLIT3_BN256 1
#endif
// rows of B one CTA loads per stage (half of BN with the CTA pair); output tile rows
// (N = 64 tiles stay single-CTA: the pair measured 10-15 % slower there)
int bn_rows(int BN, bool split3) { return split3 && gemm_pair_on() && BN >= 128 ? BN / 2 : BN; }
int bm_tile(int BN, bool split3) { return split3 && gemm_pair_on() && BN >= 128 ? 2 * BM : BM; }

int pick_bn(int64_t N, bool split3) {
    if (N <= 64) return 64;
    if (N <= 128 || (split3 && !GEMM_SPLIT3_BN256)) return 128;
    return 256;
}

}  // namespace

int launch_transpose(const float* src, int64_t rows, int64_t cols, int64_t lds, float* dst, int64_t ldd,
                     cudaStream_t s) {
    if (rows <= 0 || cols <= 0) return 0;
    if (lds % 4 == 0 && ldd % 4 == 0 && aligned16(src) && aligned16(dst)) {
        dim3 g((unsigned)((rows + 63) / 64), (unsigned)((cols + 63) / 64));
        transpose64_kernel<false><<<g, 256, 0, s>>>(src, rows, cols, lds, nullptr, dst, ldd);
        return 1;
    }
    dim3 grid((unsigned)((rows + 31) / 32), (unsigned)((cols + 31) / 32));
    transpose_kernel<<<grid, dim3(32, 8), 0, s>>>(src, rows, cols, lds, dst, ldd);
    return 1;
}

int launch_relu_transpose(const float* Z, int64_t rows, int64_t cols, int64_t ldz, float* H, float* Ht,
                          int64_t ldt, cudaStream_t s) {
    if (rows <= 0) return 0;
    if (ldz % 4 == 0 && ldt % 4 == 0 && aligned16(Z) && aligned16(H) && aligned16(Ht)) {
        dim3 g((unsigned)((rows + 63) / 64), (unsigned)((ldz + 63) / 64));
        transpose64_kernel<true><<<g, 256, 0, s>>>(Z, rows, cols, ldz, H, Ht, ldt);
        return 1;
    }
    dim3 grid((unsigned)((rows + 31) / 32), (unsigned)((ldz + 31) / 32));
    relu_transpose_kernel<<<grid, dim3(32, 8), 0, s>>>(Z, rows, cols, ldz, H, Ht, ldt);
    return 1;
}

int launch_pad_rows(const float* src, int64_t rows, int64_t cols, float* dst, int64_t ldd, cudaStream_t s) {
    const int64_t tot = rows * ldd;
    if (tot <= 0) return 0;
    pad_rows_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(src, rows, cols, dst, ldd);
    return 1;
}

// T[M x ldc] = A[M x K] (lda) · Btᵀ with Bt = Wᵀ given as [N x K] (row stride ldb)   (zero pad columns)
int gemm_tc_fwd(int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, const float* Bt, int64_t ldb, float* C,
                int64_t ldc, bool split3, cudaStream_t s) {
    const int BN = pick_bn(std::max(N, ldc), split3);
    CUtensorMap ta, tb;
    if (!make_map(&ta, A, M, K, lda, BK, BM, split3) || !make_map(&tb, Bt, N, K, ldb, BK, bn_rows(BN, split3), split3))
        CDF_FAIL(CDFGNN_ECUDA, "cuTensorMapEncodeTiled failed (fwd)");
    EpiArgs ep{C, ldc, nullptr, 0, nullptr, 0, 0, 0};
    CUtensorMap tc;
    ep.tma = make_store_map(&tc, C, M, ldc, ldc, 1, false) ? 1 : 0;
    return launch_bn<false, false>(BN, split3, ta, tb, tc, M, N, K, 1, ep, s);
}

// C[M x ldc] = (A[M x K] (lda) · Bᵀ) ⊙ 𝟙[mask > 0], B given as [N x K] (row stride ldb, K-major)
int gemm_tc_bwd_data(int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, const float* Bk, int64_t ldb,
                     float* C, int64_t ldc, const float* mask, int64_t ldm, bool split3, cudaStream_t s) {
    const int BN = pick_bn(std::max(N, ldc), split3);
    CUtensorMap ta, tb;
    if (!make_map(&ta, A, M, K, lda, BK, BM, split3) || !make_map(&tb, Bk, N, K, ldb, BK, bn_rows(BN, split3), split3))
        CDF_FAIL(CDFGNN_ECUDA, "cuTensorMapEncodeTiled failed (bwd data)");
    EpiArgs ep{C, ldc, mask, ldm, nullptr, 0, 0, 0};
    CUtensorMap tc;
    ep.tma = (!mask || (ldm & 3) == 0) && make_store_map(&tc, C, M, ldc, ldc, 1, false) ? 1 : 0;
    return launch_bn<false, false>(BN, split3, ta, tb, tc, M, N, K, 1, ep, s);
}

// C[M x N] (+)= Ht · Stᵀ with Ht = Hᵀ [M x K] (ldh) and St = Sᵀ [N x K] (lds), K = vertices; split-K
// ∇W = Hᵀ S reading H [K x M] and S [K x N] in place as MN-major operands (128-B swizzle with
// 32-B atoms, the layout the UMMA requires for MN-major tf32): no transposed copies
int gemm_tc_wgrad_mn(int64_t M, int64_t N, int64_t K, const float* H, int64_t ldh, const float* S, int64_t lds,
                     float* C, int64_t ldc, float* ws, int64_t ws_cap, bool accumulate, bool split3, cudaStream_t s,
                     int* launches) {
    const int BN = pick_bn(N, split3);
    CUtensorMap ta, tb;
    if (!make_map(&ta, H, K, M, ldh, 32, BK, split3, true) || !make_map(&tb, S, K, N, lds, 32, BK, split3, true))
        CDF_FAIL(CDFGNN_ECUDA, "cuTensorMapEncodeTiled failed (wgrad, MN-major)");
    const int64_t ldw = (N + 3) / 4 * 4;
    const int64_t tiles = ((M + bm_tile(BN, split3) - 1) / bm_tile(BN, split3)) * ((N + BN - 1) / BN);
    const int64_t total_kb = (K + BK - 1) / BK;
    int64_t splits = std::max<int64_t>(1, std::min<int64_t>((bm_tile(BN, split3) == BM ? 2 * 148 : 148) / std::max<int64_t>(tiles, 1), total_kb / 8));
    while (splits > 1 && splits * M * ldw > ws_cap) splits--;
    const int kbps = (int)((total_kb + splits - 1) / splits);
    const int zs = (int)((total_kb + kbps - 1) / kbps);
    EpiArgs ep{nullptr, 0, nullptr, 0, ws, ldw, 0, 0};
    CUtensorMap tc;
    ep.tma = make_store_map(&tc, ws, M, ldw, ldw, zs, true) ? 1 : 0;
    int rc = launch_bn<true, true>(BN, split3, ta, tb, tc, M, N, K, (int)splits, ep, s);
    if (rc != CDFGNN_OK) CDF_FAIL(rc, "wgrad launch failed");
    const int64_t tot = M * ldc;
    if (zs >= 32 && tot < 148 * 256)      // few outputs, long chains: a warp per output
        splitk_sum_warp_kernel<<<(unsigned)((tot * 32 + 255) / 256), 256, 0, s>>>(M, N, ldw, zs, ws, C, ldc, accumulate ? 1 : 0);
    else
        splitk_sum_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(M, N, ldw, zs, ws, C, ldc, accumulate ? 1 : 0);
    if (launches) *launches += 2;
    return cudaGetLastError() == cudaSuccess ? CDFGNN_OK : CDFGNN_ECUDA;
}

int gemm_tc_wgrad(int64_t M, int64_t N, int64_t K, const float* Ht, int64_t ldh, const float* St, int64_t lds,
                  float* C, int64_t ldc, float* ws, int64_t ws_cap, bool accumulate, bool split3, cudaStream_t s,
                  int* launches) {
    const int BN = pick_bn(N, split3);
    CUtensorMap ta, tb;
    if (!make_map(&ta, Ht, M, K, ldh, BK, BM, split3) || !make_map(&tb, St, N, K, lds, BK, bn_rows(BN, split3), split3))
        CDF_FAIL(CDFGNN_ECUDA, "cuTensorMapEncodeTiled failed (wgrad)");
    const int64_t ldw = (N + 3) / 4 * 4;
    const int64_t tiles = ((M + bm_tile(BN, split3) - 1) / bm_tile(BN, split3)) * ((N + BN - 1) / BN);
    const int64_t total_kb = (K + BK - 1) / BK;
    int64_t splits = std::max<int64_t>(1, std::min<int64_t>((bm_tile(BN, split3) == BM ? 2 * 148 : 148) / std::max<int64_t>(tiles, 1), total_kb / 8));
    while (splits > 1 && splits * M * ldw > ws_cap) splits--;
    const int kbps = (int)((total_kb + splits - 1) / splits);
    const int zs = (int)((total_kb + kbps - 1) / kbps);
    EpiArgs ep{nullptr, 0, nullptr, 0, ws, ldw, 0, 0};
    CUtensorMap tc;
    ep.tma = make_store_map(&tc, ws, M, ldw, ldw, zs, true) ? 1 : 0;
    int rc = launch_bn<false, false>(BN, split3, ta, tb, tc, M, N, K, (int)splits, ep, s);
    if (rc != CDFGNN_OK) CDF_FAIL(rc, "wgrad launch failed");
    const int64_t tot = M * ldc;
    if (zs >= 32 && tot < 148 * 256)      // few outputs, long chains: a warp per output
        splitk_sum_warp_kernel<<<(unsigned)((tot * 32 + 255) / 256), 256, 0, s>>>(M, N, ldw, zs, ws, C, ldc, accumulate ? 1 : 0);
    else
        splitk_sum_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(M, N, ldw, zs, ws, C, ldc, accumulate ? 1 : 0);
    if (launches) *launches += 2;
    return cudaGetLastError() == cudaSuccess ? CDFGNN_OK : CDFGNN_ECUDA;
}

}  // namespace cdfgnn
