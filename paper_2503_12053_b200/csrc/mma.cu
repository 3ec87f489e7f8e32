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
// CTA = 4 warps. The grid is (S, ceil(M/128)) with S CTAs per cluster
// splitting K. Per CTA:
//   * all 128 threads stage the B operand of the CTA's K range (16 x K_cta,
//     converted to the MMA type, 128-byte swizzled K-major) in smem once;
//   * warp 0 / lane 0 streams 16 KB A tiles (128 x 128 bytes) through an
//     NST-deep mbarrier ring with cp.async.bulk.tensor (SWIZZLE_128B);
//   * warp 1 / lane 0 issues tcgen05.mma (M = 128, N = 16, fp32 accumulator in
//     32 TMEM columns) — 4 MMAs per 16 KB tile — and tcgen05.commit frees the slot;
//   * all 4 warps read the 128 x 16 accumulator back with tcgen05.ld (warp w
//     owns TMEM lanes 32w..32w+31 = rows m0+32w..), the S partials of a cluster
//     are summed in rank order through distributed shared memory (deterministic),
//     and the epilogue applies bias + ReLU (forward) or the ReLU mask (backward).
//
// At micro-batch 16 a weight feeds 16 MACs: ~8 flop per 4-byte (tf32) or 16
// flop per 2-byte (bf16) element — far under the tensor ridge, so the kernel is
// bound by HBM bandwidth on the weight stream; the tensor cores only remove the
// SIMT issue bound.
#include "kernels.cuh"

#include <cooperative_groups.h>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstring>
#include <mutex>

namespace cg = cooperative_groups;

namespace fb200 {

namespace {

constexpr int kMmaThreads = 128;
constexpr int kTileBytes = 16384;      // A tile per pipeline stage: 128 rows x 128 bytes
constexpr int kBAtomBytes = 16 * 128;  // B operand per 128-byte K atom: 16 rows x 128 bytes
constexpr int kRedStride = 17;         // padded row of the split-K partial tile

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t addr = smem_u32(bar);
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(addr), "r"(parity)
            : "memory");
    }
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

// UMMA shared-memory descriptor (sm_100): start >> 4 [0,14), LBO >> 4 [16,30),
// SBO >> 4 [32,46), version 1 [46,48), layout [61,64): SWIZZLE_128B = 2, or
// SWIZZLE_128B_BASE32B = 1 (32-byte swizzle atoms: the only MN-major layout of tf32).
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint64_t layout = 2) {
    return static_cast<uint64_t>((addr >> 4) & 0x3FFFu) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16) |
           (static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (layout << 61);
}

__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc,
                                     bool tf32) {
    if (tf32)
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
    else
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// ES = operand bytes (4: tf32 from fp32, 2: bf16); BWD = A is MN-major (W^T).
template <int ES, bool BWD, int S>
__global__ void __cluster_dims__(S, 1, 1) __launch_bounds__(kMmaThreads, 1) mma_layer_kernel(const __grid_constant__ MmaArgs a) {
    constexpr int KA = 128 / ES;       // K elements per 128-byte atom
    constexpr int UK = 32 / ES;        // K per tcgen05.mma (32 bytes of operand)
    constexpr bool TF32 = ES == 4;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int nst = a.stages;
    unsigned char* sA = base;
    unsigned char* sB = sA + nst * kTileBytes;
    float* red = reinterpret_cast<float*>(sB + a.atoms_per_cta * kBAtomBytes);
    uint64_t* full = reinterpret_cast<uint64_t*>(red + 128 * kRedStride);
    uint64_t* empty = full + nst;
    uint64_t* done = empty + nst;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int q = S > 1 ? static_cast<int>(cg::this_cluster().block_rank()) : 0;
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
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }

    // ---- B operand: rows n < B of the CTA's K range, 16-byte chunks, swizzled
    // chunk j of row n lands at (n/8)*1024 + (n%8)*128 + ((j ^ n%8) * 16)
    {
        const int chunks = na * 16 * 8;  // atoms x rows x 16-byte chunks
        for (int e = threadIdx.x; e < chunks; e += kMmaThreads) {
            const int j = e & 7, n = (e >> 3) & 15, at = e >> 7;
            const int k0 = (a_lo + at) * KA + j * (16 / ES);
            float v[16 / ES];
#pragma unroll
            for (int i = 0; i < 16 / ES; ++i) v[i] = 0.f;
            if (n < a.N) {
                const float* row = a.X + static_cast<size_t>(a.xidx ? __ldg(a.xidx + n) : n) * a.ldx;
                if (k0 + 16 / ES <= a.K && a.vec) {
                    if constexpr (ES == 4) {
                        const float4 t = __ldg(reinterpret_cast<const float4*>(row + k0));
                        v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
                    } else {
                        const float4 t0 = __ldg(reinterpret_cast<const float4*>(row + k0));
                        const float4 t1 = __ldg(reinterpret_cast<const float4*>(row + k0 + 4));
                        v[0] = t0.x; v[1] = t0.y; v[2] = t0.z; v[3] = t0.w;
                        v[4] = t1.x; v[5] = t1.y; v[6] = t1.z; v[7] = t1.w;
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < 16 / ES; ++i)
                        if (k0 + i < a.K) v[i] = __ldg(row + k0 + i);
                }
            }
            unsigned char* dst = sB + at * kBAtomBytes + (n >> 3) * 1024 + (n & 7) * 128 + ((j ^ (n & 7)) << 4);
            if constexpr (ES == 4) {
                *reinterpret_cast<float4*>(dst) = make_float4(v[0], v[1], v[2], v[3]);
            } else {
                uint4 p;
                __nv_bfloat162 h0 = __floats2bfloat162_rn(v[0], v[1]), h1 = __floats2bfloat162_rn(v[2], v[3]);
                __nv_bfloat162 h2 = __floats2bfloat162_rn(v[4], v[5]), h3 = __floats2bfloat162_rn(v[6], v[7]);
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
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0 && lane == 0 && na > 0) {
        // ---- TMA producer
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
            mbar_wait(full + s, (i / nst) & 1);
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
            }
            umma_commit(empty + s);
        }
        umma_commit(done);
    }
    __syncwarp();

    // ---- epilogue: TMEM -> registers (thread = row m, 16 columns n)
    float acc[16];
    if (na > 0) {
        mbar_wait(done, 0);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        tmem_ld16(tmem + (static_cast<uint32_t>(warp * 32) << 16), acc);
    } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = 0.f;
    }
    const int row = threadIdx.x;  // accumulator row m0 + row

    auto finish = [&](int m, int n, float v) {
        if (m >= a.M || n >= a.N) return;
        const size_t o = static_cast<size_t>(n) * a.ldy + m;
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
        for (int n = 0; n < 16; ++n) finish(m0 + row, n, acc[n]);
    } else {
#pragma unroll
        for (int n = 0; n < 16; ++n) red[row * kRedStride + n] = acc[n];
        cg::cluster_group cl = cg::this_cluster();
        cl.sync();
        // CTA q of the cluster finishes rows [q*R, (q+1)*R), summing the S
        // partials in rank order
        constexpr int R = 128 / S;
        for (int e = threadIdx.x; e < R * 16; e += kMmaThreads) {
            const int r = q * R + (e % R), n = e / R;
            float v = 0.f;
#pragma unroll
            for (int p = 0; p < S; ++p) v += cl.map_shared_rank(red, p)[r * kRedStride + n];
            finish(m0 + r, n, v);
        }
        cl.sync();  // peers keep their smem until every partial is read
    }

    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
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

template <int ES, bool BWD, int S>
const void* mma_func(size_t smem) {
    static size_t configured = 0;  // > 48 KB dynamic smem needs an opt-in per function
    const void* f = reinterpret_cast<const void*>(&mma_layer_kernel<ES, BWD, S>);
    if (smem > configured) {
        cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        configured = smem;
    }
    return f;
}

template <int ES, bool BWD>
const void* mma_func_s(int S, size_t smem) {
    switch (S) {
        case 1: return mma_func<ES, BWD, 1>(smem);
        case 2: return mma_func<ES, BWD, 2>(smem);
        case 4: return mma_func<ES, BWD, 4>(smem);
        default: return mma_func<ES, BWD, 8>(smem);
    }
}

}  // namespace

bool mma_supported(bool bf16, int in, int out) {
    // TMA: global row stride (in x element bytes) must be a multiple of 16 bytes
    const int es = bf16 ? 2 : 4;
    return (static_cast<long long>(in) * es) % 16 == 0 && in >= 1 && out >= 1 && encode_fn() != nullptr;
}

MmaGeom mma_geom(bool bf16, bool bwd, int in, int out) {
    const int es = bf16 ? 2 : 4;
    MmaGeom g{};
    const int M = bwd ? in : out, K = bwd ? out : in;
    g.mtiles = (M + 127) / 128;
    g.katoms = static_cast<int>((static_cast<long long>(K) * es + 127) / 128);
    // ~256 CTAs (<= 2 per SM, all resident) so the weight stream has enough
    // bytes in flight; the cluster splits K and reduces through DSMEM
    int S = 1;
    while (S < 8 && g.mtiles * S * 2 <= 256 && S * 2 <= g.katoms) S *= 2;
    g.S = S;
    g.apc = (g.katoms + S - 1) / S;
    g.stages = g.apc < 4 ? g.apc : 4;
    g.smem = 1024 + static_cast<size_t>(g.stages) * kTileBytes + static_cast<size_t>(g.apc) * kBAtomBytes +
             128 * kRedStride * sizeof(float) + (2 * g.stages + 1) * 8 + 16;
    return g;
}

void spec_mma(const MmaLayer& L, KernelSpec& k) {
    const int es = L.bf16 ? 2 : 4;
    const MmaGeom g = mma_geom(L.bf16, L.bwd, L.in, L.out);
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
    a.vec = (a.ldx % 4 == 0) && ((reinterpret_cast<uintptr_t>(L.X) & 15u) == 0);
    const void* f = es == 2 ? (L.bwd ? mma_func_s<2, true>(g.S, g.smem) : mma_func_s<2, false>(g.S, g.smem))
                            : (L.bwd ? mma_func_s<4, true>(g.S, g.smem) : mma_func_s<4, false>(g.S, g.smem));
    static_assert(sizeof(MmaArgs) <= sizeof(k.arg0), "kernel argument too large");
    k.func = f;
    k.grid = dim3(g.S, g.mtiles);
    k.block = dim3(kMmaThreads);
    k.smem = g.smem;
    std::memcpy(k.arg0, &a, sizeof(MmaArgs));
    k.nargs = 1;
}

}  // namespace fb200
