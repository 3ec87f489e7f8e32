// tcgen05 / TMEM / TMA dense-layer kernels of the fast precision modes
// (FERRET_PREC_TF32, FERRET_PREC_BF16).
//
// Reference math (reference root proj/include/ferret/):
//   forward   z = W x + b, ReLU              net.hpp:99-113, learner.hpp:426-432
//   backward  prev = W^T delta, ReLU mask    learner.hpp:468-474, net.hpp:188-196
//
// One launch computes D[m][n] = sum_k A[m][k] * Bop[n][k] for one layer and
// the B <= 16 samples of a pipeline unit:
//   forward:  m = output row r, k = input column c, A = W     (K-major: W rows are contiguous in c)
//             Bop = the unit's input rows x_b (K-major)
//   backward: m = input column c, k = output row r, A = W^T   (MN-major: W rows are contiguous in m)
//             Bop = the unit's deltas delta_b (K-major)
// so the weight matrix is streamed from HBM exactly once per launch, by TMA,
// in its stored row-major layout, with no transposed copy.
//
// CTA = 4 warps. The grid is (S, ceil(M/128)), S CTAs splitting K. Per CTA:
//   * all 128 threads stage the B operand of the CTA's K range (16 x K_cta,
//     converted to the MMA type, 128-byte swizzled K-major) in smem once;
//   * warp 0 / lane 0 streams 16 KB A tiles (128 x 128 bytes) through an
//     NST-deep mbarrier ring with cp.async.bulk.tensor (SWIZZLE_128B);
//   * warp 1 / lane 0 issues tcgen05.mma (M = 128, N = 16, fp32 accumulator in
//     32 TMEM columns) — 4 MMAs per 16 KB tile — and tcgen05.commit frees the slot;
//   * all 4 warps read the 128 x 16 accumulator back with tcgen05.ld (warp w
//     owns TMEM lanes 32w..32w+31 = rows m0+32w..); with S > 1 the partial tile
//     goes to L2 scratch and the last CTA of the M tile sums the S partials in
//     split order (deterministic), then applies bias + ReLU (forward) or the
//     ReLU mask (backward).
// The grid is sized to one wave of one CTA per SM with the deepest A ring the
// shared memory holds (the first version used 8-CTA clusters and a DSMEM
// reduction: cluster residency capped it at 120 co-resident CTAs, two waves,
// 21 % of HBM bandwidth — profiles/README.md).
//
// At micro-batch 16 a weight feeds 16 MACs: ~8 flop per 4-byte (tf32) or 16
// flop per 2-byte (bf16) element — far under the tensor ridge, so the kernel is
// bound by HBM bandwidth on the weight stream; the tensor cores only remove the
// SIMT issue bound.
#include "kernels.cuh"
#include "umma.cuh"

#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

namespace fb200 {

namespace {

constexpr int kMmaThreads = 320;  // warp 0 TMA, warp 1 MMA, warps 2-9 stage B; warps 2-5 run the epilogue
constexpr int kStagers = 256;
constexpr int kTileBytes = 16384;      // A tile per pipeline stage: 128 rows x 128 bytes
constexpr int kBAtomBytes = 16 * 128;  // B operand per 128-byte K atom: 16 rows x 128 bytes
constexpr size_t kMaxSmem = 225 * 1024;  // opt-in dynamic shared memory per CTA (227 KB less static)


// Epilogue of the dense-layer kernels, warps 2-5: TMEM -> registers (warp w reads TMEM
// lanes of quadrant w % 4: thread = accumulator row m0 + row, 16 columns n), then bias +
// ReLU (forward) or the ReLU mask (backward); with S > 1 K splits the partial tile goes
// to L2 scratch and the last CTA of the M tile sums the S partials in split order.
// STACK: the accumulator is two 16-column halves to add (3xTF32 with B hi / lo stacked as
// one N = 32 operand: columns 0-15 = hi.hi + lo.hi, columns 16-31 = hi.lo).
template <bool BWD, bool STACK = false>
__device__ __forceinline__ void mma_epilogue(const MmaArgs& a, uint32_t tmem, uint64_t* done, bool any, int warp,
                                             int lane, int m0, int q, int S) {
    const int row = (warp & 3) * 32 + lane;
    float acc[16];
    if (any) {
        mbar_wait(done, 0);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t taddr = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
        tmem_ld16(taddr, acc);
        if constexpr (STACK) {
            float hl[16];
            tmem_ld16(taddr + 16, hl);
#pragma unroll
            for (int i = 0; i < 16; ++i) acc[i] += hl[i];
        }
    } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = 0.f;
    }
    auto finish = [&](int m, int nn, float v) {
        if (m >= a.M || nn >= a.N) return;
        const size_t o = static_cast<size_t>(nn) * a.ldy + m;
        if (!BWD) {
            v += __ldg(a.bias + m);
            if (a.relu) v = v > 0.f ? v : 0.f;
        } else if (a.mask) {
            v = __ldg(a.mask + o) > 0.f ? v : 0.f;
        }
        a.Y[o] = v;
    };
    if (S == 1) {
#pragma unroll
        for (int nn = 0; nn < 16; ++nn) finish(m0 + row, nn, acc[nn]);
        return;
    }
    // split-K: partial tile to global scratch ([n][128], coalesced); the last CTA of the
    // M tile to arrive sums the S partials in split order (deterministic) and runs the
    // epilogue
    float* part = a.partial + (static_cast<size_t>(blockIdx.y) * S + q) * 128 * 16;
#pragma unroll
    for (int nn = 0; nn < 16; ++nn) part[nn * 128 + row] = acc[nn];
    __threadfence();
    asm volatile("bar.sync 1, 128;" ::: "memory");  // the 4 epilogue warps
    __shared__ unsigned last;
    if (warp == 2 && lane == 0) last = atomicAdd(a.counters + blockIdx.y, 1u) == static_cast<unsigned>(S - 1);
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (!last) return;
    __threadfence();
    // sum in split order; this CTA's own partial is still in registers, the others'
    // 16 values per split are loaded together
    const float* base = a.partial + static_cast<size_t>(blockIdx.y) * S * 128 * 16 + row;
    float v[16];
#pragma unroll
    for (int nn = 0; nn < 16; ++nn) v[nn] = 0.f;
    for (int p = 0; p < S; ++p) {
        float tv[16];
        if (p == q) {
#pragma unroll
            for (int nn = 0; nn < 16; ++nn) tv[nn] = acc[nn];
        } else {
#pragma unroll
            for (int nn = 0; nn < 16; ++nn) tv[nn] = __ldcg(base + (static_cast<size_t>(p) * 16 + nn) * 128);
        }
#pragma unroll
        for (int nn = 0; nn < 16; ++nn) v[nn] += tv[nn];
    }
#pragma unroll
    for (int nn = 0; nn < 16; ++nn) finish(m0 + row, nn, v[nn]);
    if (warp == 2 && lane == 0) a.counters[blockIdx.y] = 0u;  // self-resetting (graph replays)
}

template <int ES, bool BWD, bool SPLIT = false>
__global__ void __launch_bounds__(kMmaThreads, 1) mma_layer_kernel(const __grid_constant__ MmaArgs a) {
    FB_PDL_ENTRY();
    constexpr int KA = 128 / ES;       // K elements per 128-byte atom
    constexpr int UK = 32 / ES;        // K per tcgen05.mma (32 bytes of operand)
    constexpr bool TF32 = ES == 4;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int nst = a.stages;
    unsigned char* sA = base;
    unsigned char* sAlo = sA + nst * kTileBytes;                 // SPLIT: lo parts of the A ring
    unsigned char* sB = sAlo + (SPLIT ? nst * kTileBytes : 0);
    unsigned char* sBlo = sB + a.atoms_per_cta * kBAtomBytes;    // SPLIT: lo parts of B
    uint64_t* full = reinterpret_cast<uint64_t*>(sBlo + (SPLIT ? a.atoms_per_cta * kBAtomBytes : 0));
    uint64_t* empty = full + nst;
    uint64_t* done = empty + nst;
    uint64_t* bready = done + 1;  // per B atom: staged by the stager warps
    uint64_t* lready = bready + a.atoms_per_cta;  // SPLIT, per ring stage: A split into hi / lo
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(lready + (SPLIT ? nst : 0));

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int S = a.splits, q = blockIdx.x;
    // optional phase timestamps (globaltimer ns) per CTA: start, setup done,
    // B staged, first A tile landed, accumulator done, exit
    unsigned long long* stamp = a.stamps ? a.stamps + (static_cast<size_t>(blockIdx.y) * gridDim.x + blockIdx.x) * 8 : nullptr;
    auto tick = [&](int k) {
        if (stamp) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            stamp[k] = t;
        }
    };
    if (threadIdx.x == 0) tick(0);
    const int m0 = blockIdx.y * 128;
    const int a_lo = q * a.atoms_per_cta;
    const int a_hi = min(a.katoms, a_lo + a.atoms_per_cta);
    const int na = max(0, a_hi - a_lo);

    if (threadIdx.x == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&a.tmap)) : "memory");
        for (int s = 0; s < nst; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        mbar_init(done, 1);
        for (int i = 0; i < na; ++i) mbar_init(bready + i, kStagers);
        if (SPLIT)
            for (int s = 0; s < nst; ++s) mbar_init(lready + s, kStagers);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    if (threadIdx.x == 0) tick(1);

    if (warp == 0 && lane == 0 && na > 0) {
        // ---- TMA producer: one 16 KB A tile per ring stage
        for (int i = 0; i < na; ++i) {
            const int s = i % nst;
            if (i >= nst) mbar_wait(empty + s, ((i / nst) - 1) & 1);
            mbar_expect_tx(full + s, kTileBytes);
            unsigned char* dst = sA + s * kTileBytes;
            const int kk = (a_lo + i) * KA;
            if (!BWD) {
                tma_load_2d(dst, &a.tmap, full + s, kk, m0);  // {K inner, M rows}: 128 rows x 128 bytes
            } else {
#pragma unroll
                for (int c = 0; c < 128 / KA; ++c)  // {M inner, K rows}: (128/KA) boxes of KA rows x 128 bytes
                    tma_load_2d(dst + c * KA * 128, &a.tmap, full + s, m0 + c * KA, kk);
            }
        }
    } else if (warp == 1 && lane == 0 && na > 0) {
        // ---- MMA issuer: D[128 x 16] += A[128 x KA] * B[16 x KA]^T per tile
        // instruction descriptor: D f32, A/B tf32 (2) or bf16 (1), A major, N >> 3, M >> 4
        const uint32_t fmt = TF32 ? 2u : 1u;
        const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((BWD ? 1u : 0u) << 15) | ((16u >> 3) << 17) |
                               ((128u >> 4) << 24);
        for (int i = 0; i < na; ++i) {
            const int s = i % nst;
            mbar_wait(bready + i, 0);
            mbar_wait(SPLIT ? lready + s : full + s, (i / nst) & 1);
            if (i == 0) tick(3);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t abase = smem_u32(sA + s * kTileBytes);
            const uint32_t bbase = smem_u32(sB + i * kBAtomBytes);
#pragma unroll
            for (int k = 0; k < KA / UK; ++k) {
                // K-major A: advance 32 bytes inside the swizzled row; SBO = 8 rows x 128 B.
                // MN-major A: K step = UK rows of 128 B; LBO = next 128-byte column of M (KA rows
                // down); SBO = the next group of 8 K rows (bf16, 16-byte swizzle atoms) or of
                // 4 K rows (tf32, 32-byte swizzle atoms).
                const uint64_t ad = BWD ? (TF32 ? smem_desc(abase + k * UK * 128, KA * 128, 512, 1)
                                                : smem_desc(abase + k * UK * 128, KA * 128, 1024))
                                        : smem_desc(abase + k * 32, 16, 1024);
                const uint64_t bd = smem_desc(bbase + k * 32, 16, 1024);
                umma(tmem, ad, bd, idesc, (i > 0 || k > 0) ? 1u : 0u, TF32);
                if constexpr (SPLIT) {  // + hi_A lo_B + lo_A hi_B
                    const uint32_t lofs = static_cast<uint32_t>(sAlo - sA);
                    const uint32_t blofs = static_cast<uint32_t>(sBlo - sB);
                    const uint64_t bdl = smem_desc(bbase + blofs + k * 32, 16, 1024);
                    const uint64_t adl = BWD ? smem_desc(abase + lofs + k * UK * 128, KA * 128, 512, 1)
                                             : smem_desc(abase + lofs + k * 32, 16, 1024);
                    umma(tmem, ad, bdl, idesc, 1u, TF32);
                    umma(tmem, adl, bd, idesc, 1u, TF32);
                }
            }
            umma_commit(empty + s);
        }
        umma_commit(done);
    } else if (warp >= 2) {
        // ---- B operand, staged by warps 2-9 while A streams: rows n < N of the
        // CTA's K range as 16-byte chunks, swizzled: chunk j of row n lands at
        // (n/8)*1024 + (n%8)*128 + ((j ^ n%8) * 16). Rows n >= N stay unwritten
        // (D column n depends on B row n only; those columns are never stored).
        // Thread t owns chunk column j = t % 8 of row n = (t / 8) % 16 in atoms
        // t / 128, t / 128 + 2, ... of each round of G atoms, so its row pointer
        // is resolved once and a round's U loads have no dependence on each
        // other; each staged atom is published on its mbarrier after a proxy fence.
        constexpr int CE = 16 / ES, G = 16, U = G * 128 / kStagers;  // elements/chunk, atoms/round, chunks/thread
        const int t = threadIdx.x - 64, j = t & 7, n = (t >> 3) & 15, ao = t >> 7;
        const bool rowv = n < a.N;
        const float* rowp = rowv ? a.X + static_cast<size_t>(a.xidx ? __ldg(a.xidx + n) : n) * a.ldx : a.X;
        for (int g0 = 0; g0 < na; g0 += G) {
            float v[U][CE];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int at = g0 + ao + 2 * u;
                const int k0 = (a_lo + at) * KA + j * CE;
                const float* src = rowp + k0;
                if (at < na && rowv && a.vec && k0 + CE <= a.K) {
#pragma unroll
                    for (int c = 0; c < CE / 4; ++c) {
                        const float4 x4 = __ldg(reinterpret_cast<const float4*>(src) + c);
                        v[u][4 * c] = x4.x; v[u][4 * c + 1] = x4.y; v[u][4 * c + 2] = x4.z; v[u][4 * c + 3] = x4.w;
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < CE; ++i) v[u][i] = (at < na && rowv && k0 + i < a.K) ? __ldg(src + i) : 0.f;
                }
            }
            if (rowv) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int at = g0 + ao + 2 * u;
                    if (at >= na) continue;
                    unsigned char* dst = sB + at * kBAtomBytes + (n >> 3) * 1024 + (n & 7) * 128 + ((j ^ (n & 7)) << 4);
                    if constexpr (ES == 4) {
                        if constexpr (SPLIT) {
                            const float4 hi = make_float4(tf32_hi(v[u][0]), tf32_hi(v[u][1]), tf32_hi(v[u][2]),
                                                          tf32_hi(v[u][3]));
                            *reinterpret_cast<float4*>(dst) = hi;
                            *reinterpret_cast<float4*>(dst + (sBlo - sB)) =
                                make_float4(v[u][0] - hi.x, v[u][1] - hi.y, v[u][2] - hi.z, v[u][3] - hi.w);
                        } else {
                            *reinterpret_cast<float4*>(dst) = make_float4(v[u][0], v[u][1], v[u][2], v[u][3]);
                        }
                    } else {
                        uint4 p;
                        __nv_bfloat162 h0 = __floats2bfloat162_rn(v[u][0], v[u][1]), h1 = __floats2bfloat162_rn(v[u][2], v[u][3]);
                        __nv_bfloat162 h2 = __floats2bfloat162_rn(v[u][4], v[u][5]), h3 = __floats2bfloat162_rn(v[u][6], v[u][7]);
                        p.x = *reinterpret_cast<uint32_t*>(&h0);
                        p.y = *reinterpret_cast<uint32_t*>(&h1);
                        p.z = *reinterpret_cast<uint32_t*>(&h2);
                        p.w = *reinterpret_cast<uint32_t*>(&h3);
                        *reinterpret_cast<uint4*>(dst) = p;
                    }
                }
            }
            // generic-proxy smem writes -> visible to the tensor core (async proxy)
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            for (int at = g0; at < min(na, g0 + G); ++at)
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bready + at)) : "memory");
        }
        if (threadIdx.x == 64) tick(2);
        if constexpr (SPLIT) {
            // split every landed A tile in place: hi (low 13 mantissa bits cleared)
            // stays in the ring slot, lo goes to the parallel slot (elementwise, so
            // the swizzled layout is preserved); published per stage on lready
            for (int i = 0; i < na; ++i) {
                const int s = i % nst;
                mbar_wait(full + s, (i / nst) & 1);
                float4* A4 = reinterpret_cast<float4*>(sA + s * kTileBytes);
                float4* L4 = reinterpret_cast<float4*>(sAlo + s * kTileBytes);
                for (int e = t; e < kTileBytes / 16; e += kStagers) {
                    // hi stays implicit (kind::tf32 drops the low 13 mantissa bits of the raw operand)
                    const float4 x = A4[e];
                    const float4 hi = make_float4(tf32_hi(x.x), tf32_hi(x.y), tf32_hi(x.z), tf32_hi(x.w));
                    L4[e] = make_float4(x.x - hi.x, x.y - hi.y, x.z - hi.z, x.w - hi.w);
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(lready + s)) : "memory");
            }
        }
    }
    __syncwarp();

    // ---- epilogue, warps 2-5
    if (warp >= 2 && warp < 6) {
        if (warp == 2 && lane == 0 && na > 0) {
            mbar_wait(done, 0);
            tick(4);
        }
        mma_epilogue<BWD>(a, tmem, done, na > 0, warp, lane, m0, q, S);
    }

    if (warp == 2 && lane == 0) tick(5);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
    }
}

// ---------------------------------------------------------------------------
// mma_ring_kernel: the dense layer with the B operand staged per ring stage
// instead of for the CTA's whole K range up front (mma_layer_kernel), so the
// first MMA waits for one A tile, not for the whole B slice, and the ring is as
// deep as the A stream needs. A ring stage holds the TMA'd A tile (16 KB) and the
// unit's B atom (2 KB); in the fp32 parity mode (SPLIT, 3xTF32, see tf32_hi) also
// the A tile's lo part (16 KB, hi stays implicit: kind::tf32 drops the low
// mantissa bits) and B as hi + lo: 36 KB. Two CTAs per SM. Roles:
//   warp 0 / lane 0  TMA producer: A tile of stage s once the MMA freed it (empty[s])
//   warp 1 / lane 0  MMA issuer: per stage KA/UK k-steps x 1 MMA (SPLIT: 2, hi_A x
//                    [B hi; B lo] as one N = 32 operand, then lo_A x B hi), commit -> empty[s]
//   warps 2-9        stagers: load the unit's B atom i (L2) before waiting for the
//                    A tile, convert / split it into the stage (and split A for
//                    SPLIT), publish the stage on lready[s]; warps 2-5 then run the
//                    epilogue
// (the whole-K B staging left the fp32 parity mode room for 2 stages of one CTA:
// 1.5 TB/s on config 5's 4096 x 4096 layers; this kernel: 2.5 TB/s forward)
// ---------------------------------------------------------------------------
template <int ES, bool SPLIT>
__host__ __device__ constexpr int ring_stage_bytes() { return (SPLIT ? 2 : 1) * (kTileBytes + kBAtomBytes); }

template <int ES, bool BWD, bool SPLIT>
__global__ void __launch_bounds__(kMmaThreads, 2) mma_ring_kernel(const __grid_constant__ MmaArgs a) {
    FB_PDL_ENTRY();
    constexpr int KA = 128 / ES, UK = 32 / ES;  // K elements per 128-byte atom / per tcgen05.mma
    constexpr bool TF32 = ES == 4;
    constexpr int SB = ring_stage_bytes<ES, SPLIT>();
    constexpr int BOFF = (SPLIT ? 2 : 1) * kTileBytes;  // B hi inside a stage (B lo follows)
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int nst = a.stages;
    auto stage = [&](int s) { return base + static_cast<size_t>(s) * SB; };
    uint64_t* full = reinterpret_cast<uint64_t*>(stage(nst));
    uint64_t* empty = full + nst;
    uint64_t* lready = empty + nst;
    uint64_t* done = lready + nst;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int S = a.splits, q = blockIdx.x;
    const int m0 = blockIdx.y * 128;
    const int a_lo = q * a.atoms_per_cta;
    const int a_hi = min(a.katoms, a_lo + a.atoms_per_cta);
    const int na = max(0, a_hi - a_lo);
    // optional phase timestamps (globaltimer ns) per CTA: 0 start, 1 setup done, 2 first A
    // tile landed, 3 first MMA issued, 4 accumulator done, 5 exit, 6 last TMA issued,
    // 7 epilogue done
    unsigned long long* stamp = a.stamps ? a.stamps + (static_cast<size_t>(blockIdx.y) * gridDim.x + blockIdx.x) * 8 : nullptr;
    auto tick = [&](int idx) {
        if (stamp) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            stamp[idx] = t;
        }
    };
    if (threadIdx.x == 0) tick(0);

    if (threadIdx.x == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&a.tmap)) : "memory");
        for (int s = 0; s < nst; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
            mbar_init(lready + s, kStagers);
        }
        mbar_init(done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    if (threadIdx.x == 0) tick(1);

    if (warp == 0 && lane == 0 && na > 0) {
        for (int i = 0; i < na; ++i) {
            const int s = i % nst;
            if (i >= nst) mbar_wait(empty + s, ((i / nst) - 1) & 1);
            mbar_expect_tx(full + s, kTileBytes);
            unsigned char* dst = stage(s);
            const int kk = (a_lo + i) * KA;
            if (!BWD) {
                tma_load_2d(dst, &a.tmap, full + s, kk, m0);  // {K inner, M rows}: 128 rows x 128 bytes
            } else {
#pragma unroll
                for (int c = 0; c < 128 / KA; ++c)  // {M inner, K rows}: (128/KA) boxes of KA rows x 128 bytes
                    tma_load_2d(dst + c * KA * 128, &a.tmap, full + s, m0 + c * KA, kk);
            }
        }
        tick(6);
    } else if (warp == 1 && lane == 0 && na > 0) {
        // D f32, A/B tf32 (2) or bf16 (1), A K-major (forward) or MN-major (backward), N = 16, M = 128
        const uint32_t fmt = TF32 ? 2u : 1u;
        const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((BWD ? 1u : 0u) << 15) | ((16u >> 3) << 17) |
                               ((128u >> 4) << 24);
        // SPLIT: B hi (rows 0-15) and B lo (rows 16-31) are one N = 32 operand, so hi_A meets
        // both in one MMA (A read once for hi.hi + hi.lo); lo.hi is an N = 16 MMA into columns 0-15
        const uint32_t idesc32 = (idesc & ~(0x3Fu << 17)) | ((32u >> 3) << 17);
        for (int i = 0; i < na; ++i) {
            const int s = i % nst;
            mbar_wait(lready + s, (i / nst) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            if (i == 0) tick(3);
            const uint32_t ah = smem_u32(stage(s)), bh = ah + BOFF;
#pragma unroll
            for (int k = 0; k < KA / UK; ++k) {
                // K-major A: advance 32 bytes inside the swizzled row; SBO = 8 rows x 128 B.
                // MN-major A: K step = UK rows of 128 B; LBO = the next 128-byte column of M
                // (KA rows down); SBO = the next group of 8 K rows (bf16, 16-byte swizzle
                // atoms) or of 4 K rows (tf32, 32-byte swizzle atoms).
                auto adesc = [&](uint32_t at) {
                    return BWD ? (TF32 ? smem_desc(at + k * UK * 128, KA * 128, 512, 1)
                                       : smem_desc(at + k * UK * 128, KA * 128, 1024))
                               : smem_desc(at + k * 32, 16, 1024);
                };
                const uint64_t bdh = smem_desc(bh + k * 32, 16, 1024);
                if constexpr (SPLIT) {
                    umma(tmem, adesc(ah), bdh, idesc32, (i > 0 || k > 0) ? 1u : 0u, true);
                    umma(tmem, adesc(ah + kTileBytes), bdh, idesc, 1u, true);
                } else {
                    umma(tmem, adesc(ah), bdh, idesc, (i > 0 || k > 0) ? 1u : 0u, TF32);
                }
            }
            umma_commit(empty + s);
        }
        umma_commit(done);
    } else if (warp >= 2) {
        // B atom: 16 rows x 128 bytes; thread t < 128 owns 16-byte chunk j = t % 8 of row
        // n = t / 8 (swizzled to (n/8)*1024 + (n%8)*128 + ((j ^ n%8) * 16)), i.e. CE = 16/ES
        // consecutive K elements; for SPLIT the A tile's 1024 float4 are split by all 256
        constexpr int CE = 16 / ES;
        const int t = threadIdx.x - 64, j = t & 7, n = t >> 3;
        const bool bthr = t < 128, rowv = bthr && n < a.N;
        const float* rowp = rowv ? a.X + static_cast<size_t>(a.xidx ? __ldg(a.xidx + n) : n) * a.ldx : a.X;
        const int boff = (n >> 3) * 1024 + (n & 7) * 128 + ((j ^ (n & 7)) << 4);
        struct BV {
            float v[CE];
        };
        auto load_b = [&](int i) {
            BV r;
#pragma unroll
            for (int e = 0; e < CE; ++e) r.v[e] = 0.f;
            const int k0 = (a_lo + i) * KA + j * CE;
            if (rowv && i < na) {
                const float* src = rowp + k0;
                if (a.vec && k0 + CE <= a.K) {
#pragma unroll
                    for (int c = 0; c < CE / 4; ++c) {
                        const float4 x4 = __ldg(reinterpret_cast<const float4*>(src) + c);
                        r.v[4 * c] = x4.x; r.v[4 * c + 1] = x4.y; r.v[4 * c + 2] = x4.z; r.v[4 * c + 3] = x4.w;
                    }
                } else {
#pragma unroll
                    for (int e = 0; e < CE; ++e) r.v[e] = k0 + e < a.K ? __ldg(src + e) : 0.f;
                }
            }
            return r;
        };
        BV bnext = load_b(0);
        for (int i = 0; i < na; ++i) {
            const int s = i % nst;
            const BV bv = bnext;
            bnext = load_b(i + 1);  // the next atom's B is in flight while this stage is prepared
            mbar_wait(full + s, (i / nst) & 1);
            if (i == 0 && t == 0) tick(2);
            unsigned char* st = stage(s);
            if constexpr (SPLIT) {
                const float4* A4 = reinterpret_cast<const float4*>(st);
                float4* L4 = reinterpret_cast<float4*>(st + kTileBytes);
#pragma unroll
                for (int e = t; e < kTileBytes / 16; e += kStagers) {
                    const float4 x = A4[e];
                    L4[e] = make_float4(x.x - tf32_hi(x.x), x.y - tf32_hi(x.y), x.z - tf32_hi(x.z), x.w - tf32_hi(x.w));
                }
            }
            if (bthr) {  // rows n >= N stay stale: D column n reads B row n only, never stored
                unsigned char* dst = st + BOFF + boff;
                if constexpr (ES == 4) {
                    if constexpr (SPLIT) {
                        const float4 hi = make_float4(tf32_hi(bv.v[0]), tf32_hi(bv.v[1]), tf32_hi(bv.v[2]), tf32_hi(bv.v[3]));
                        *reinterpret_cast<float4*>(dst) = hi;
                        *reinterpret_cast<float4*>(dst + kBAtomBytes) =
                            make_float4(bv.v[0] - hi.x, bv.v[1] - hi.y, bv.v[2] - hi.z, bv.v[3] - hi.w);
                    } else {
                        *reinterpret_cast<float4*>(dst) = make_float4(bv.v[0], bv.v[1], bv.v[2], bv.v[3]);
                    }
                } else {
                    uint4 p;
                    __nv_bfloat162 h0 = __floats2bfloat162_rn(bv.v[0], bv.v[1]), h1 = __floats2bfloat162_rn(bv.v[2], bv.v[3]);
                    __nv_bfloat162 h2 = __floats2bfloat162_rn(bv.v[4], bv.v[5]), h3 = __floats2bfloat162_rn(bv.v[6], bv.v[7]);
                    p.x = *reinterpret_cast<uint32_t*>(&h0);
                    p.y = *reinterpret_cast<uint32_t*>(&h1);
                    p.z = *reinterpret_cast<uint32_t*>(&h2);
                    p.w = *reinterpret_cast<uint32_t*>(&h3);
                    *reinterpret_cast<uint4*>(dst) = p;
                }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(lready + s)) : "memory");
        }
    }
    __syncwarp();
    if (warp >= 2 && warp < 6) {
        if (warp == 2 && lane == 0 && na > 0) {
            mbar_wait(done, 0);
            tick(4);
        }
        mma_epilogue<BWD, SPLIT>(a, tmem, done, na > 0, warp, lane, m0, q, S);
        if (warp == 2 && lane == 0) tick(7);
    }

    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) tick(5);
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
    }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

template <int ES, bool BWD, bool SPLIT = false>
const void* mma_func(size_t smem) {
    static size_t configured = 0;  // > 48 KB dynamic smem needs an opt-in per function
    const void* f = reinterpret_cast<const void*>(&mma_layer_kernel<ES, BWD, SPLIT>);
    if (smem > configured) {
        cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        configured = smem;
    }
    return f;
}

template <int ES, bool BWD, bool SPLIT>
const void* ring_func(size_t smem) {
    static size_t configured = 0;
    const void* f = reinterpret_cast<const void*>(&mma_ring_kernel<ES, BWD, SPLIT>);
    if (smem > configured) {
        cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        configured = smem;
    }
    return f;
}

// mma_ring_kernel unless FERRET_MMA_WHOLE_B=1 (A/B knob: mma_layer_kernel, B staged for the whole K range)
bool ring_b() {
    static const bool on = !std::getenv("FERRET_MMA_WHOLE_B") || std::atoi(std::getenv("FERRET_MMA_WHOLE_B")) == 0;
    return on;
}

}  // namespace

bool mma_supported(bool bf16, int in, int out) {
    // TMA: global row stride (in x element bytes) must be a multiple of 16 bytes
    const int es = bf16 ? 2 : 4;
    return (static_cast<long long>(in) * es) % 16 == 0 && in >= 1 && out >= 1 && encode_fn() != nullptr;
}

MmaGeom mma_geom(bool bf16, bool bwd, int in, int out, bool split) {
    const int es = bf16 ? 2 : 4;
    if (ring_b()) {
        // mma_ring_kernel: two CTAs per SM, ring stages of A (+ A lo) and one B atom (hi, lo)
        const int sb = split ? ring_stage_bytes<4, true>() : ring_stage_bytes<4, false>();
        MmaGeom g{};
        const int M = bwd ? in : out, K = bwd ? out : in;
        g.mtiles = (M + 127) / 128;
        g.katoms = static_cast<int>((static_cast<long long>(K) * es + 127) / 128);
        // K splits: about 96 CTAs per layer (two thirds of the SMs at one CTA each), not the one full
        // wave of two CTAs per SM that an isolated launch prefers: inside the concurrent chunk graph a
        // layer shares the GPU with update kernels and other stages' layers, and the smaller grid left
        // them room — C5 fp32 +2.5 % over the full wave (S = 9 -> 3 at 4096 outputs;
        // profiles/r2/split_bench.txt)
        int S = 96 / g.mtiles;
        if (S > 16) S = 16;
        if (S > g.katoms) S = g.katoms;
        if (S < 1) S = 1;
        if (const char* env = std::getenv("FERRET_MMA_SPLIT")) S = std::atoi(env);  // experiment knob
        g.apc = (g.katoms + S - 1) / S;
        g.S = (g.katoms + g.apc - 1) / g.apc;
        constexpr size_t kPerCta = 113 * 1024;  // two CTAs per SM (228 KB less the per-CTA reserve)
        const size_t fixed = 1024 + 4 * 16 * 8 + 16;
        g.stages = static_cast<int>((kPerCta - fixed) / static_cast<size_t>(sb));
        if (g.stages > g.apc) g.stages = g.apc;
        if (g.stages > 16) g.stages = 16;
        g.smem = fixed + static_cast<size_t>(g.stages) * static_cast<size_t>(sb);
        g.partial_floats = g.S > 1 ? static_cast<size_t>(g.mtiles) * g.S * 128 * 16 : 0;
        return g;
    }
    const int mult = split ? 2 : 1;  // 3xTF32: hi + lo copies of the A ring and of B
    MmaGeom g{};
    const int M = bwd ? in : out, K = bwd ? out : in;
    g.mtiles = (M + 127) / 128;
    g.katoms = static_cast<int>((static_cast<long long>(K) * es + 127) / 128);
    // one wave of one CTA per SM: the K splits of an M tile are separate CTAs
    // (partials reduced through L2 by the last one), every CTA streams its A
    // slice through the deepest TMA ring its shared memory holds
    int S = 148 / g.mtiles;
    if (S > 16) S = 16;
    if (S > g.katoms) S = g.katoms;
    if (S < 1) S = 1;
    if (const char* env = std::getenv("FERRET_MMA_SPLIT")) S = std::atoi(env);  // experiment knob
    g.apc = (g.katoms + S - 1) / S;
    g.S = (g.katoms + g.apc - 1) / g.apc;  // every split owns >= 1 atom
    const size_t fixed = 1024 + static_cast<size_t>(g.apc) * (mult * kBAtomBytes + 8) + 256 + 64;
    g.stages = static_cast<int>((kMaxSmem - fixed) / (mult * kTileBytes));
    if (g.stages > g.apc) g.stages = g.apc;
    if (g.stages > 16) g.stages = 16;
    g.smem = fixed + static_cast<size_t>(g.stages) * mult * kTileBytes;
    g.partial_floats = g.S > 1 ? static_cast<size_t>(g.mtiles) * g.S * 128 * 16 : 0;
    return g;
}

void spec_mma(const MmaLayer& L, KernelSpec& k) {
    const int es = L.bf16 ? 2 : 4;
    const bool split = L.split && !L.bf16;
    const MmaGeom g = mma_geom(L.bf16, L.bwd, L.in, L.out, split);
    MmaArgs a{};
    // tensor map of W (out x in, row-major): dims {in, out}; boxes of 128 bytes x rows
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(L.in), static_cast<cuuint64_t>(L.out)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(L.in) * es};
    const int ka = 128 / es;
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(ka), static_cast<cuuint32_t>(L.bwd ? ka : 128)};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_fn()(&a.tmap, es == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                                   const_cast<void*>(L.W), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                   (L.bwd && es == 4) ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        std::fprintf(stderr, "ferret-b200: cuTensorMapEncodeTiled failed (%d)\n", static_cast<int>(r));
        std::abort();
    }
    a.bias = L.bias;
    a.X = L.X;
    a.xidx = L.xidx;
    a.mask = L.mask;
    a.Y = L.Y;
    a.M = L.bwd ? L.in : L.out;
    a.K = L.bwd ? L.out : L.in;
    a.N = L.B;
    a.ldx = a.K;
    a.ldy = a.M;
    a.katoms = g.katoms;
    a.atoms_per_cta = g.apc;
    a.stages = g.stages;
    a.relu = L.relu;
    a.splits = g.S;
    a.partial = L.partial;
    a.counters = L.counters;
    a.stamps = L.stamps;
    if (g.S > 1 && (!L.partial || !L.counters)) {
        std::fprintf(stderr, "ferret-b200: split-K dense layer without scratch\n");
        std::abort();
    }
    a.vec = (a.ldx % 4 == 0) && ((reinterpret_cast<uintptr_t>(L.X) & 15u) == 0);
    const void* f;
    if (ring_b())
        f = es == 2 ? (L.bwd ? ring_func<2, true, false>(g.smem) : ring_func<2, false, false>(g.smem))
          : split   ? (L.bwd ? ring_func<4, true, true>(g.smem) : ring_func<4, false, true>(g.smem))
                    : (L.bwd ? ring_func<4, true, false>(g.smem) : ring_func<4, false, false>(g.smem));
    else
        f = es == 2 ? (L.bwd ? mma_func<2, true>(g.smem) : mma_func<2, false>(g.smem))
          : split   ? (L.bwd ? mma_func<4, true, true>(g.smem) : mma_func<4, false, true>(g.smem))
                    : (L.bwd ? mma_func<4, true>(g.smem) : mma_func<4, false>(g.smem));
    static_assert(sizeof(MmaArgs) <= sizeof(k.arg0), "kernel argument too large");
    k.func = f;
    k.grid = dim3(g.S, g.mtiles);
    k.block = dim3(kMmaThreads);
    k.smem = g.smem;
    std::memcpy(k.arg0, &a, sizeof(MmaArgs));
    k.nargs = 1;
}

}  // namespace fb200
