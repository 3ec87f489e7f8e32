// sm_100a kernels of the ferret-b200 pipelined stream trainer.
//
// Reference math restated here (reference root proj/include/ferret/):
//   fwd_kernel        affine_forward + apply_activation      net.hpp:99-113, learner.hpp:426-432
//   head_kernel       softmax / argmax / softmax-CE delta    net.hpp:115-125,150-154, learner.hpp:443-447
//   bwd_kernel        ReLU mask + prev = W^T delta           learner.hpp:456-474, net.hpp:178-196
//   update_kernel     gW = delta (x) x, Compensator::apply,  learner.hpp:460-467,491-504,97-120
//                     mean, SGD step, new version slot       compensate.hpp:42-130
//   normalize_kernel  RunningNormalizer observe + apply      stream.hpp:312-328
// All fp32 except the normalizer (fp64, bit-exact with the host).
#include "kernels.cuh"

#include <cuda_bf16.h>

#include <cfloat>
#include <cstdio>
#include <cstdlib>
#include <cstring>

namespace fb200 {

namespace {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__host__ __device__ __forceinline__ bool aligned16(const void* p) {
    return (reinterpret_cast<uintptr_t>(p) & 15u) == 0;
}

// Reduce NV per-lane values across the warp with NV*log2(32/NV) + NV-1
// shuffles (transpose-reduce): afterwards lane L holds the warp sum of value
// index (L % NV). NV is a power of two <= 32.
template <int NV>
__device__ __forceinline__ float warp_transpose_sum(float (&v)[NV], int lane) {
#pragma unroll
    for (int o = 16; o >= NV; o >>= 1)
#pragma unroll
        for (int j = 0; j < NV; ++j) v[j] += __shfl_xor_sync(0xffffffffu, v[j], o);
#pragma unroll
    for (int o = NV / 2; o >= 1; o >>= 1) {
        const bool upper = (lane & o) != 0;
#pragma unroll
        for (int j = 0; j < o; ++j) {
            const float send = upper ? v[j] : v[j + o];
            const float keep = upper ? v[j + o] : v[j];
            v[j] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    return v[0];
}

// softmax head of sample b over logits z (net.hpp:115-125,150-154, learner.hpp:443-447),
// one warp: first-index argmax (mode 0) or scale * (softmax - onehot) (mode 1)
__device__ __forceinline__ void head_sample(const float* z, int n_out, int mode, int label, int* pred_b, float* d,
                                            float scale, int lane) {
    // max with first-index tie break
    float best = -FLT_MAX;
    int best_k = 0x7fffffff;
    for (int k = lane; k < n_out; k += 32) {
        const float v = z[k];
        if (v > best || (v == best && k < best_k)) {
            best = v;
            best_k = k;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int ok = __shfl_xor_sync(0xffffffffu, best_k, o);
        if (ov > best || (ov == best && ok < best_k)) {
            best = ov;
            best_k = ok;
        }
    }
    if (mode == 0) {
        if (lane == 0) *pred_b = best_k;
        return;
    }
    float sum = 0.f;
    for (int k = lane; k < n_out; k += 32) sum += expf(z[k] - best);
    sum = warp_sum(sum);
    for (int k = lane; k < n_out; k += 32) {
        const float p = expf(z[k] - best) / sum;
        d[k] = scale * (k == label ? p - 1.f : p);
    }
}

// ---------------------------------------------------------------------------
// forward: CTA = `groups` row groups x `nwk` K-slices (groups * nwk = 8 warps).
// A warp accumulates RW rows x B samples over its K slice (float4 when the
// rows are 16-byte aligned), transpose-reduces them, and the CTA sums the K
// slices in smem, adds the bias and applies ReLU.
// ---------------------------------------------------------------------------
template <int BT, int RW, bool VEC>
__global__ void __launch_bounds__(kThreads) fwd_kernel(const FwdArgs a, int nwk) {
    FB_PDL_ENTRY();
    constexpr int NV = RW * BT;
    __shared__ float part[kWarps][NV];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int groups = kWarps / nwk;
    const int g = warp / nwk, kw = warp % nwk;
    const int r0 = (blockIdx.x * groups + g) * RW;
    const int nk = VEC ? (a.in >> 2) : a.in;
    const int kc = (nk + nwk - 1) / nwk;
    const int k_lo = kw * kc, k_hi = min(nk, k_lo + kc);
    const int B = a.B;
    // input row b starts at X + xrow(b) (replay gathers rows from the pool);
    // offsets resolved once, before the K loop
    size_t xo[BT];
#pragma unroll
    for (int b = 0; b < BT; ++b) xo[b] = (size_t)(b < B ? (a.xidx ? __ldg(a.xidx + b) : b) : 0) * a.in;
    auto xrow = [&](int b) -> size_t { return xo[b]; };
    float acc[RW][BT];
#pragma unroll
    for (int i = 0; i < RW; ++i)
#pragma unroll
        for (int b = 0; b < BT; ++b) acc[i][b] = 0.f;
    if (r0 < a.out) {
        // the B input values of this K position are loaded once and reused by
        // the RW weight rows; each weight load is reused by the B samples
        for (int k = k_lo + lane; k < k_hi; k += 32) {
            if (VEC) {
                float4 xv[BT];
#pragma unroll
                for (int b = 0; b < BT; ++b)
                    xv[b] = b < B ? __ldg(reinterpret_cast<const float4*>(a.X + xrow(b)) + k)
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int i = 0; i < RW; ++i) {
                    if (r0 + i >= a.out) break;
                    const float4 w = __ldg(reinterpret_cast<const float4*>(a.W + (size_t)(r0 + i) * a.in) + k);
#pragma unroll
                    for (int b = 0; b < BT; ++b) {
                        acc[i][b] = fmaf(w.x, xv[b].x, acc[i][b]);
                        acc[i][b] = fmaf(w.y, xv[b].y, acc[i][b]);
                        acc[i][b] = fmaf(w.z, xv[b].z, acc[i][b]);
                        acc[i][b] = fmaf(w.w, xv[b].w, acc[i][b]);
                    }
                }
            } else {
                float xv[BT];
#pragma unroll
                for (int b = 0; b < BT; ++b) xv[b] = b < B ? __ldg(a.X + xrow(b) + k) : 0.f;
#pragma unroll
                for (int i = 0; i < RW; ++i) {
                    if (r0 + i >= a.out) break;
                    const float w = __ldg(a.W + (size_t)(r0 + i) * a.in + k);
#pragma unroll
                    for (int b = 0; b < BT; ++b) acc[i][b] = fmaf(w, xv[b], acc[i][b]);
                }
            }
        }
    }
    // transpose-reduce in chunks of 32 values: lane L ends with value c*32 + L
    constexpr int NC = NV > 32 ? NV / 32 : 1;
    constexpr int NW = NV > 32 ? 32 : NV;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        float flat[NW];
#pragma unroll
        for (int q = 0; q < NW; ++q) {
            const int idx = c * NW + q;
            flat[q] = acc[idx / BT][idx % BT];
        }
        const float s = warp_transpose_sum<NW>(flat, lane);
        if (lane < NW) part[warp][c * NW + lane] = s;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < groups * NV; t += kThreads) {
        const int gg = t / NV, idx = t % NV;
        const int i = idx / BT, b = idx % BT;
        const int r = (blockIdx.x * groups + gg) * RW + i;
        if (r >= a.out || b >= B) continue;
        float z = 0.f;
        for (int q = 0; q < nwk; ++q) z += part[gg * nwk + q][idx];
        z += a.bias[r];
        if (a.relu) z = z > 0.f ? z : 0.f;
        a.Y[(size_t)b * a.out + r] = z;
    }
    if (a.head_mode >= 0) {  // one CTA wrote every logit: the head in the same launch
        __syncthreads();
        for (int b = warp; b < B; b += kWarps)
            head_sample(a.Y + (size_t)b * a.out, a.out, a.head_mode, a.head_mode == 0 ? 0 : a.labels[b],
                        a.pred ? a.pred + b : nullptr, a.delta ? a.delta + (size_t)b * a.out : nullptr, a.scale, lane);
    }
}

template <class Args>
void fill(KernelSpec& k, const void* func, dim3 grid, dim3 block, const Args& a) {
    static_assert(sizeof(Args) <= sizeof(k.arg0), "kernel argument too large");
    k.func = func;
    k.grid = grid;
    k.block = block;
    k.smem = 0;
    std::memcpy(k.arg0, &a, sizeof(Args));
    k.nargs = 1;
}

int fwd_rows_per_cta(int in, bool vec, int RW) {
    const int nk = vec ? (in >> 2) : in;
    int nwk = (nk + 63) / 64;
    nwk = nwk >= 8 ? 8 : nwk >= 4 ? 4 : nwk >= 2 ? 2 : 1;
    return (kWarps / nwk) * RW;
}

template <int BT, int RW>
void fwd_spec(const FwdArgs& a, bool vec, KernelSpec& k) {
    const int nk = vec ? (a.in >> 2) : a.in;
    int nwk = (nk + 63) / 64;  // >= 2 K-units per lane per warp
    nwk = nwk >= 8 ? 8 : nwk >= 4 ? 4 : nwk >= 2 ? 2 : 1;
    const int rows_per_cta = (kWarps / nwk) * RW;
    const int grid = (a.out + rows_per_cta - 1) / rows_per_cta;
    const void* f = vec ? reinterpret_cast<const void*>(&fwd_kernel<BT, RW, true>)
                        : reinterpret_cast<const void*>(&fwd_kernel<BT, RW, false>);
    fill(k, f, dim3(grid), dim3(kThreads), a);
    k.arg1 = nwk;
    k.nargs = 2;
}

// ---------------------------------------------------------------------------
// softmax head: one warp per sample.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) head_kernel(const HeadArgs a) {
    FB_PDL_ENTRY();
    const int lane = threadIdx.x & 31;
    const int b = blockIdx.x * kWarps + (threadIdx.x >> 5);
    if (b >= a.B) return;
    const int label = a.mode == 0 ? 0 : a.labels[a.lidx ? a.lidx[b] : b];
    head_sample(a.logits + (size_t)b * a.n_out, a.n_out, a.mode, label, a.pred ? a.pred + b : nullptr,
                a.delta ? a.delta + (size_t)b * a.n_out : nullptr, a.scale, lane);
}

// ---------------------------------------------------------------------------
// backward delta propagation: CTA = column tile (32 lanes x V columns) x row
// split; warps take interleaved rows of the split, the CTA sums the warps in
// a fixed order in smem; with several row splits the last CTA of a column
// tile reduces the split partials in split order (deterministic).
// ---------------------------------------------------------------------------
constexpr int kBwdMaxRows = 512;   // rows per split (delta staging in smem)

// Small layers (out <= 256): latency, not bandwidth, bounds the node. One CTA
// per 32 columns, every row of the layer: each warp loads its 32 rows of the
// column strip in one trip (32 independent loads in flight per lane), the 8
// warps reduce once through smem and the CTA writes d_in directly — no split
// partials, no second global round trip.
constexpr int kBwdSmallRows = 256;

template <int BT>
__global__ void __launch_bounds__(kThreads) bwd_small_kernel(const BwdArgs a) {
    FB_PDL_ENTRY();
    __shared__ __align__(16) float sd[kBwdSmallRows][BT];
    __shared__ float part[kWarps][BT][33];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = blockIdx.x * 32 + lane;
    const int B = a.B, out = a.out;
    for (int i = threadIdx.x; i < BT * out; i += kThreads) {
        const int b = i / out, r = i - b * out;
        sd[r][b] = b < B ? a.d_out[(size_t)b * out + r] : 0.f;
    }
    float w[kBwdSmallRows / kWarps];
    constexpr int RPW = kBwdSmallRows / kWarps;  // rows per warp
#pragma unroll
    for (int q = 0; q < RPW; ++q) {
        const int r = warp + q * kWarps;
        w[q] = (r < out && c < a.in) ? __ldg(a.W + (size_t)r * a.in + c) : 0.f;
    }
    __syncthreads();
    float acc[BT];
#pragma unroll
    for (int b = 0; b < BT; ++b) acc[b] = 0.f;
#pragma unroll
    for (int q = 0; q < RPW; ++q) {
        const int r = warp + q * kWarps;
        if (r >= out) break;
#pragma unroll
        for (int b = 0; b < BT; b += (BT % 4 == 0 ? 4 : 1)) {
            if (BT % 4 == 0) {
                const float4 d = *reinterpret_cast<const float4*>(&sd[r][b]);
                acc[b] = fmaf(w[q], d.x, acc[b]);
                acc[(b + 1) % BT] = fmaf(w[q], d.y, acc[(b + 1) % BT]);
                acc[(b + 2) % BT] = fmaf(w[q], d.z, acc[(b + 2) % BT]);
                acc[(b + 3) % BT] = fmaf(w[q], d.w, acc[(b + 3) % BT]);
            } else {
                acc[b] = fmaf(w[q], sd[r][b], acc[b]);
            }
        }
    }
#pragma unroll
    for (int b = 0; b < BT; ++b) part[warp][b][lane] = acc[b];
    __syncthreads();
    for (int i = threadIdx.x; i < B * 32; i += kThreads) {
        const int b = i >> 5, cc = i & 31, col = blockIdx.x * 32 + cc;
        if (col >= a.in) continue;
        float v = 0.f;
#pragma unroll
        for (int q = 0; q < kWarps; ++q) v += part[q][b][cc];
        if (a.mask && !(a.mask[(size_t)b * a.in + col] > 0.f)) v = 0.f;
        a.d_in[(size_t)b * a.in + col] = v;
    }
}

template <int BT, int V>
__global__ void __launch_bounds__(kThreads) bwd_kernel(const BwdArgs a) {
    FB_PDL_ENTRY();
    // deltas as [row][sample]: one row's B values are read as float4s
    __shared__ __align__(16) float sd[kBwdMaxRows][BT];
    extern __shared__ float wpart[];  // [kWarps][BT][32 * V] per-warp partials (dynamic)
    __shared__ bool last_cta;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int splits = gridDim.y;
    const int rows_per = (a.out + splits - 1) / splits;
    const int rs = blockIdx.y * rows_per, re = min(a.out, rs + rows_per);
    const int B = a.B;
    const int c0 = blockIdx.x * 32 * V + lane * V;
    for (int i = threadIdx.x; i < BT * rows_per; i += kThreads) {
        const int b = i / rows_per, rr = i % rows_per;
        sd[rr][b] = (b < B && rs + rr < re) ? a.d_out[(size_t)b * a.out + rs + rr] : 0.f;
    }
    __syncthreads();
    // acc[b][v] += w[v] * delta(row, b), delta read 4 samples at a time
    auto row_fma = [&](const float (&w)[V], int rr, float (&acc)[BT][V]) {
        if (BT % 4 == 0) {
#pragma unroll
            for (int b = 0; b < BT; b += 4) {
                const float4 d = *reinterpret_cast<const float4*>(&sd[rr][b]);
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    acc[b][v] = fmaf(w[v], d.x, acc[b][v]);
                    acc[(b + 1) % BT][v] = fmaf(w[v], d.y, acc[(b + 1) % BT][v]);
                    acc[(b + 2) % BT][v] = fmaf(w[v], d.z, acc[(b + 2) % BT][v]);
                    acc[(b + 3) % BT][v] = fmaf(w[v], d.w, acc[(b + 3) % BT][v]);
                }
            }
        } else {
#pragma unroll
            for (int b = 0; b < BT; ++b) {
                const float d = sd[rr][b];
#pragma unroll
                for (int v = 0; v < V; ++v) acc[b][v] = fmaf(w[v], d, acc[b][v]);
            }
        }
    };
    float acc[BT][V];
#pragma unroll
    for (int b = 0; b < BT; ++b)
#pragma unroll
        for (int v = 0; v < V; ++v) acc[b][v] = 0.f;
    if (c0 < a.in) {
        // RU rows per trip with independent loads in flight (the rows are
        // L2/HBM latency-bound, not bandwidth-bound, at these sizes)
        constexpr int RU = 4;
        int r = rs + warp;
        for (; r + (RU - 1) * kWarps < re; r += RU * kWarps) {
            float w[RU][V];
#pragma unroll
            for (int q = 0; q < RU; ++q) {
                const float* wp = a.W + (size_t)(r + q * kWarps) * a.in + c0;
                if (V == 4) {
                    const float4 w4 = __ldg(reinterpret_cast<const float4*>(wp));
                    w[q][0] = w4.x; w[q][1 % V] = w4.y; w[q][2 % V] = w4.z; w[q][3 % V] = w4.w;
                } else {
                    w[q][0] = __ldg(wp);
                }
            }
#pragma unroll
            for (int q = 0; q < RU; ++q) row_fma(w[q], r + q * kWarps - rs, acc);
        }
        for (; r < re; r += kWarps) {
            float w[V];
            if (V == 4) {
                const float4 w4 = __ldg(reinterpret_cast<const float4*>(a.W + (size_t)r * a.in + c0));
                w[0] = w4.x; w[1 % V] = w4.y; w[2 % V] = w4.z; w[3 % V] = w4.w;
            } else {
                w[0] = __ldg(a.W + (size_t)r * a.in + c0);
            }
            row_fma(w, r - rs, acc);
        }
    }
    // cross-warp sum: every warp parks its partials, one barrier, then each
    // thread sums its (sample, column) pairs over the warps in warp order
    constexpr int TC = 32 * V;
#pragma unroll
    for (int b = 0; b < BT; ++b)
#pragma unroll
        for (int v = 0; v < V; ++v) wpart[(warp * BT + b) * TC + lane * V + v] = acc[b][v];
    __syncthreads();
    auto sacc_at = [&](int b, int cc) {
        float s = 0.f;
#pragma unroll
        for (int q = 0; q < kWarps; ++q) s += wpart[(q * BT + b) * TC + cc];
        return s;
    };
    const int tile0 = blockIdx.x * 32 * V;
    if (splits == 1) {
        for (int i = threadIdx.x; i < B * 32 * V; i += kThreads) {
            const int b = i / (32 * V), cc = i % (32 * V), c = tile0 + cc;
            if (c >= a.in) continue;
            float val = sacc_at(b, cc);
            if (a.mask && !(a.mask[(size_t)b * a.in + c] > 0.f)) val = 0.f;
            a.d_in[(size_t)b * a.in + c] = val;
        }
        return;
    }
    for (int i = threadIdx.x; i < B * 32 * V; i += kThreads) {
        const int b = i / (32 * V), cc = i % (32 * V), c = tile0 + cc;
        if (c < a.in) a.partial[((size_t)blockIdx.y * B + b) * a.in + c] = sacc_at(b, cc);
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last_cta = atomicAdd(&a.counters[blockIdx.x], 1u) == (unsigned)(splits - 1);
    __syncthreads();
    if (!last_cta) return;
    __threadfence();
    for (int i = threadIdx.x; i < B * 32 * V; i += kThreads) {
        const int b = i / (32 * V), cc = i % (32 * V), c = tile0 + cc;
        if (c >= a.in) continue;
        const float* p = a.partial + (size_t)b * a.in + c;
        const size_t stride = (size_t)B * a.in;
        float val = 0.f;
        int sp = 0;
        for (; sp + 4 <= splits; sp += 4) {
            const float p0 = __ldcg(p + sp * stride), p1 = __ldcg(p + (sp + 1) * stride),
                        p2 = __ldcg(p + (sp + 2) * stride), p3 = __ldcg(p + (sp + 3) * stride);
            val += p0;
            val += p1;
            val += p2;
            val += p3;
        }
        for (; sp < splits; ++sp) val += __ldcg(p + sp * stride);
        if (a.mask && !(a.mask[(size_t)b * a.in + c] > 0.f)) val = 0.f;
        a.d_in[(size_t)b * a.in + c] = val;
    }
    if (threadIdx.x == 0) a.counters[blockIdx.x] = 0u;
}

// ---------------------------------------------------------------------------
// compensation of one element for one pending gradient (compensate.hpp).
// vers[i] is the base of chain version i; the chain is vers[first .. last]
// (vers[last] is the live version, whose value at element e is th_cur).
// ---------------------------------------------------------------------------
struct ElemState {
    float ld, vr, va, gp;
};

// ---------------------------------------------------------------------------
// iter_fisher arithmetic (compensate.hpp:82-104) with every rounding spelled out (explicit
// fma / mul / add, no compiler-chosen contraction), shared by every update kernel — single,
// tiled, float4, smem-streamed and grouped — so they all produce the same bits.
// ---------------------------------------------------------------------------
// the lambda / v_r / v_a step (compensate.hpp:87-95); d0 = theta_1 - theta_0; returns lambda
__device__ __forceinline__ float iter_learn(float g, float d0, float& ld, float& vr, float& va, float lam_base,
                                            float alpha, float eta, float nu) {
    const float one_m_a = __fsub_rn(1.f, alpha);
    float lam = __fadd_rn(lam_base, ld);
    const float dv = __fmul_rn(one_m_a, __fsub_rn(g, vr));
    const float resid = __fmaf_rn(-lam, va, dv);
    const float grad_l = __fmaf_rn(__fmul_rn(-2.f, resid), va, __fmul_rn(__fmul_rn(2.f, nu), lam));
    ld = __fmaf_rn(-eta, grad_l, ld);
    lam = __fadd_rn(lam_base, ld);
    vr = __fmaf_rn(alpha, vr, __fmul_rn(one_m_a, g));
    va = __fmaf_rn(alpha, va, __fmul_rn(__fmul_rn(__fmul_rn(one_m_a, g), g), d0));
    return lam;
}
// one step of the fold: out += lambda * out^2 * (theta_{s+1} - theta_s)   compensate.hpp:99-102
__device__ __forceinline__ float iter_fold(float o, float lam, float d) {
    return __fmaf_rn(__fmul_rn(__fmul_rn(lam, o), o), d, o);
}
// theta_new = theta_cur - step * out   learner.hpp:497-502
__device__ __forceinline__ float sgd_new(float cur, float step, float o) { return __fmaf_rn(-step, o, cur); }

template <int POLICY>
__device__ __forceinline__ float compensate_elem(float g, const float* const* vers, int first, int last, size_t e,
                                                 float th_cur, ElemState& st, float lam_base, float alpha,
                                                 float eta, float nu, bool learn) {
    const int tau = last - first;
    if (POLICY == 0) {  // none
        return g;
    } else if (POLICY == 1) {  // step: g * 1/(1+tau)              compensate.hpp:107-113
        return g * (1.f / (1.f + (float)tau));
    } else if (POLICY == 2) {  // gap                               compensate.hpp:117-130, learner.hpp:104-111
        const float read = tau ? __ldg(vers[first] + e) : th_cur;
        const float gapv = fabsf(th_cur - read);
        const float mg = fmaxf(st.gp, 1e-12f);
        const float o = g / (1.f + gapv / mg);
        st.gp = 0.99f * st.gp + 0.01f * gapv;
        return o;
    } else if (POLICY == 3) {  // fisher: g + lambda0 g^2 (cur - read)   compensate.hpp:42-51
        const float read = tau ? __ldg(vers[first] + e) : th_cur;
        return g + lam_base * g * g * (th_cur - read);
    } else {  // iter_fisher                                            compensate.hpp:82-104
        float lam = lam_base + st.ld;
        float prev = tau >= 1 ? __ldg(vers[first] + e) : th_cur;
        if (learn && tau >= 1) {
            const float nxt = tau == 1 ? th_cur : __ldg(vers[first + 1] + e);
            lam = iter_learn(g, nxt - prev, st.ld, st.vr, st.va, lam_base, alpha, eta, nu);
        }
        float o = g;
        for (int s = first; s < last; ++s) {
            const float nxt = (s + 1 == last) ? th_cur : __ldg(vers[s + 1] + e);
            o = iter_fold(o, lam, nxt - prev);
            prev = nxt;
        }
        return o;
    }
}

// ---------------------------------------------------------------------------
// fused update: one thread per work item (V consecutive parameters of one
// weight row, or one bias), grid-stride over the stage's segments.
// ---------------------------------------------------------------------------
constexpr int kRegChain = 12;  // chain versions the iter_fisher fold keeps in registers
// iter_fisher K = 1 chains longer than this take the smem-staged update_stream_kernel
constexpr int kStreamMinChain = 16;
constexpr int kStreamMinChainLarge = 4;  // the same for stages of >= 8 M parameters (HBM-bound)

// iter_fisher (compensate.hpp:82-104) for one element with the chain values
// already in registers: cv[i] = version i (i < last), th = version `last`.
// Loops are fully unrolled and predicated so every cv[] index is static.
template <int V>
__device__ __forceinline__ float fold_iter_cached(float g, const float (&cv)[kRegChain + 1][V], int v, int first,
                                                  int last, float th, ElemState& st, float lam_base, float alpha,
                                                  float eta, float nu, bool learn) {
    float lam = lam_base + st.ld;
    if (learn && last - first >= 1) {
        float v0 = 0.f, v1 = 0.f;
#pragma unroll
        for (int i = 0; i < kRegChain; ++i)
            if (i == first) {
                v0 = cv[i][v];
                v1 = (i + 1 < last) ? cv[i + 1][v] : th;
            }
        lam = iter_learn(g, v1 - v0, st.ld, st.vr, st.va, lam_base, alpha, eta, nu);
    }
    float o = g;
#pragma unroll
    for (int i = 0; i < kRegChain; ++i)
        if (i >= first && i < last) {
            const float nxt = (i + 1 < last) ? cv[i + 1][v] : th;
            o = iter_fold(o, lam, nxt - cv[i][v]);
        }
    return o;
}

// ---------------------------------------------------------------------------
// tiled update: one parameter per thread. A CTA covers up to 8 rows x 256
// columns of one layer; the deltas of those rows (K pending x B samples) are
// staged in smem and broadcast, and with one pending gradient the unit's B
// input values of the thread's column stay in registers across the rows.
// Chain versions are read coalesced across the CTA (consecutive columns).
// ---------------------------------------------------------------------------
template <int POLICY, int BT>
__global__ void __launch_bounds__(kThreads) update_tile_kernel(const UpdArgs a) {
    FB_PDL_ENTRY();
    __shared__ float sdel[kMaxPending * kMaxBatch * kUpdMaxTileRows];
    const UpdTile t = a.tiles[blockIdx.x];
    const UpdSeg sg = a.segs[t.seg];
    const int K = a.K, B = a.B, R = t.nrows;
    const int tid = threadIdx.x;
    const int last = a.nv - 1;
    const bool learn = a.eta > 0.f && a.v_r != nullptr;
    const bool cached = POLICY == 4 && last <= kRegChain;
    if (!sg.bias && sg.g_off < 0) {
        for (int i = tid; i < K * B * R; i += kThreads) {
            const int k = i / (B * R), rem = i - k * B * R, b = rem / R, rr = rem - b * R;
            sdel[i] = __ldg(a.pend[k].stash + sg.dlt_off + (size_t)b * sg.out + t.r0 + rr);
        }
    }
    __syncthreads();
    // the element's new value, compensator state and write-back
    auto apply = [&](size_t e, int row_in_tile, int c) {
        const float th = __ldg(a.vers[last] + e);
        ElemState st{0.f, 0.f, 0.f, 0.f};
        if (POLICY == 4) {
            st.ld = a.lam_d[e];
            if (learn) {
                st.vr = a.v_r[e];
                st.va = a.v_a[e];
            }
        }
        if (POLICY == 2) st.gp = a.gap[e];
        float cv[kRegChain + 1][1];
        if (cached) {
#pragma unroll
            for (int i = 0; i < kRegChain; ++i) cv[i][0] = i < last ? __ldg(a.vers[i] + e) : 0.f;
            cv[kRegChain][0] = 0.f;
        }
        float mean = 0.f;
        for (int k = 0; k < K; ++k) {
            float g = 0.f;
            if (sg.g_off >= 0) {  // materialised gradient (convolutions: conv_wgrad / conv_bgrad)
                g = __ldg(a.pend[k].stash + sg.g_off +
                          (sg.bias ? (size_t)row_in_tile : (size_t)(t.r0 + row_in_tile) * sg.in + c));
            } else if (sg.bias) {
                const float* dl = a.pend[k].stash + sg.dlt_off + row_in_tile;  // row_in_tile = absolute row here
#pragma unroll
                for (int b = 0; b < BT; ++b)
                    if (b < B) g += __ldg(dl + (size_t)b * sg.out);
            } else {
                const float* sd = sdel + (size_t)k * B * R + row_in_tile;
                const UpdPending& pk = a.pend[k];
#pragma unroll
                for (int b = 0; b < BT; ++b) {
                    if (b >= B) break;
                    const float* xr = sg.xin_off >= 0 ? pk.stash + sg.xin_off + (size_t)b * sg.in
                                      : a.x0idx       ? pk.x0 + (size_t)__ldg(a.x0idx + b) * a.x0_ld
                                                      : pk.x0 + (size_t)b * a.x0_ld;
                    g = fmaf(sd[b * R], __ldg(xr + c), g);
                }
            }
            if (cached)
                mean += fold_iter_cached<1>(g, cv, 0, a.pend[k].first, last, th, st, a.lambda0, a.alpha, a.eta, a.nu,
                                            learn);
            else
                mean += compensate_elem<POLICY>(g, a.vers, a.pend[k].first, last, e, th, st, a.lambda0, a.alpha, a.eta,
                                                a.nu, learn);
        }
        const float nv = sgd_new(th, a.step, mean);
        a.dst[e] = nv;
        if (a.dst16) reinterpret_cast<__nv_bfloat16*>(a.dst16)[e] = __float2bfloat16_rn(nv);
        if (POLICY == 4) {
            a.lam_d[e] = st.ld;
            if (learn) {
                a.v_r[e] = st.vr;
                a.v_a[e] = st.va;
            }
        }
        if (POLICY == 2) a.gap[e] = st.gp;
    };
    if (sg.bias) {
        if (tid < R) apply((size_t)sg.elem0 + t.r0 + tid, t.r0 + tid, 0);
        return;
    }
    const int c = t.c0 + tid;
    if (c >= sg.in) return;
    for (int i = 0; i < R; ++i) apply((size_t)sg.elem0 + (size_t)(t.r0 + i) * sg.in + c, i, c);
}

// ---------------------------------------------------------------------------
// iter_fisher with one pending gradient (accumulation count 1, the default
// config): the chain is versions 0..NV-1 of the launch's table, so the fold
// length is a compile-time constant and every loop is straight-line code.
// One parameter per thread; the unit's B input values of the thread's column
// stay in registers across the tile's rows; deltas are broadcast from smem.
// ---------------------------------------------------------------------------
template <int BT, int NV>
__global__ void __launch_bounds__(kThreads) update_iter1_kernel(const UpdArgs a) {
    // Programmatic chain (trainer.cpp, FERRET_UPDATE_PDL): this launch may start while the
    // previous update of the stage still runs. Everything that update does not write — the work
    // record, the unit's deltas and inputs, versions 0 .. NV-2 of the chain — is loaded before
    // griddepcontrol.wait; the newest version and the compensator state (its outputs) after it.
    // launch_dependents follows the wait, so the next update of the stage launches only once
    // this one's own predecessor has completed (its pre-wait reads then see finished versions).
    // Latency-shaped: after the one dependent load of the CTA's work record,
    // every load of the launch — the unit's deltas (to smem), its input values
    // of the thread's column, and the version chain + compensator state of the
    // first RB rows — is issued before any arithmetic, so the kernel costs ~two
    // L2 round trips rather than one per row and stage of the address chain.
    // rows whose chains are held in registers at once (4 rows up to 12 versions measured 20 %
    // slower on C2: register pressure against the concurrent DAG, profiles/r2/update_rb_ab.txt)
    constexpr int RB = NV <= 8 ? 4 : 2;
    __shared__ float sdel[kMaxBatch * kUpdMaxTileRows];
    const UpdWork w = a.works[blockIdx.x];
    const int B = a.B, R = w.nrows, tid = threadIdx.x;
    const bool learn = a.eta > 0.f && a.v_r != nullptr;
    const UpdPending& pk = a.pend[0];
    // the fold of one element (compensate.hpp:87-102) from values in registers
    auto fold = [&](size_t e, float g, const float (&cv)[NV], float ld, float vr, float va) {
        float lam = a.lambda0 + ld;
        if (NV >= 2 && learn) {
            lam = iter_learn(g, cv[NV >= 2 ? 1 : 0] - cv[0], ld, vr, va, a.lambda0, a.alpha, a.eta, a.nu);
            a.v_r[e] = vr;
            a.v_a[e] = va;
            a.lam_d[e] = ld;
        }
        float o = g;
#pragma unroll
        for (int s = 0; s + 1 < NV; ++s) o = iter_fold(o, lam, cv[s + 1] - cv[s]);
        const float nv = sgd_new(cv[NV - 1], a.step, o);
        a.dst[e] = nv;
        if (a.dst16) reinterpret_cast<__nv_bfloat16*>(a.dst16)[e] = __float2bfloat16_rn(nv);
    };
    auto load = [&](size_t e, float (&cv)[NV], float& ld, float& vr, float& va) {
#pragma unroll
        for (int i = 0; i < NV; ++i) cv[i] = __ldg(a.vers[i] + e);
        ld = a.lam_d[e];
        vr = learn ? a.v_r[e] : 0.f;
        va = learn ? a.v_a[e] : 0.f;
    };
    // the first batch: older versions before the dependency wait, the newest + state after it
    auto load_old = [&](size_t e, float (&cv)[NV]) {
#pragma unroll
        for (int i = 0; i + 1 < NV; ++i) cv[i] = __ldg(a.vers[i] + e);
    };
    auto load_new = [&](size_t e, float (&cv)[NV], float& ld, float& vr, float& va) {
        cv[NV - 1] = a.vers[NV - 1][e];  // (not __ldg: written by the upstream update)
        ld = a.lam_d[e];
        vr = learn ? a.v_r[e] : 0.f;
        va = learn ? a.v_a[e] : 0.f;
    };
    auto dep_wait = [] {
        asm volatile("griddepcontrol.wait;" ::: "memory");
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    };
    const bool gm = w.g_off >= 0;  // materialised gradient (convolutions)
    if (w.bias) {
        if (tid >= R) {
            dep_wait();
            return;
        }
        const int r = w.r0 + tid;
        const size_t e = (size_t)w.elem0 + r;
        float cv[NV], ld, vr, va;
        load_old(e, cv);
        dep_wait();
        load_new(e, cv, ld, vr, va);
        float g = 0.f;
        if (gm) {
            g = __ldg(pk.stash + w.g_off + r);
        } else {
            const float* dl = pk.stash + w.dlt_off + r;
#pragma unroll
            for (int b = 0; b < BT; ++b)
                if (b < B) g += __ldg(dl + (size_t)b * w.out);
        }
        fold(e, g, cv, ld, vr, va);
        return;
    }
    const int c = w.c0 + tid;
    const bool live = c < w.in;
    float cv[RB][NV], ld[RB], vr[RB], va[RB];
#pragma unroll
    for (int i = 0; i < RB; ++i)
        if (live && i < R) load_old((size_t)w.elem0 + (size_t)(w.r0 + i) * w.in + c, cv[i]);
    float xv[BT];
    if (!gm) {
        for (int i = tid; i < B * R; i += kThreads) {
            const int b = i / R, rr = i - b * R;
            sdel[i] = __ldg(pk.stash + w.dlt_off + (size_t)b * w.out + w.r0 + rr);
        }
#pragma unroll
        for (int b = 0; b < BT; ++b) {
            const float* xr = w.xin_off >= 0 ? pk.stash + w.xin_off + (size_t)b * w.in
                              : a.x0idx      ? pk.x0 + (size_t)__ldg(a.x0idx + b) * a.x0_ld
                                             : pk.x0 + (size_t)b * a.x0_ld;
            xv[b] = (b < B && live) ? __ldg(xr + c) : 0.f;
        }
    }
    dep_wait();
#pragma unroll
    for (int i = 0; i < RB; ++i)
        if (live && i < R) load_new((size_t)w.elem0 + (size_t)(w.r0 + i) * w.in + c, cv[i], ld[i], vr[i], va[i]);
    __syncthreads();
    if (!live) return;
    auto grad = [&](int i) {
        if (gm) return __ldg(pk.stash + w.g_off + (size_t)(w.r0 + i) * w.in + c);
        float g = 0.f;
#pragma unroll
        for (int b = 0; b < BT; ++b) g = fmaf(sdel[b * R + i], xv[b], g);
        return g;
    };
    // rows in batches of RB, double-buffered: the loads of batch g + 1 are issued before the
    // folds of batch g, so each batch costs one L2 round trip overlapped with the previous fold
    // (not one per row); FERRET_UPDATE_PIPELINE=0 keeps the row-serial tail (experiment knob)
    if (a.pipe) {
        float nv_[RB][NV], nl[RB], nr[RB], na[RB];
        for (int g0 = 0; g0 < R; g0 += RB) {
            const int g1 = g0 + RB;
#pragma unroll
            for (int i = 0; i < RB; ++i)
                if (g1 + i < R) load((size_t)w.elem0 + (size_t)(w.r0 + g1 + i) * w.in + c, nv_[i], nl[i], nr[i], na[i]);
#pragma unroll
            for (int i = 0; i < RB; ++i)
                if (g0 + i < R)
                    fold((size_t)w.elem0 + (size_t)(w.r0 + g0 + i) * w.in + c, grad(g0 + i), cv[i], ld[i], vr[i], va[i]);
#pragma unroll
            for (int i = 0; i < RB; ++i) {
#pragma unroll
                for (int q = 0; q < NV; ++q) cv[i][q] = nv_[i][q];
                ld[i] = nl[i];
                vr[i] = nr[i];
                va[i] = na[i];
            }
        }
        return;
    }
#pragma unroll
    for (int i = 0; i < RB; ++i)
        if (i < R) fold((size_t)w.elem0 + (size_t)(w.r0 + i) * w.in + c, grad(i), cv[i], ld[i], vr[i], va[i]);
    for (int i = RB; i < R; ++i) {  // rows beyond the register batch
        const size_t e = (size_t)w.elem0 + (size_t)(w.r0 + i) * w.in + c;
        float cr[NV], l0, r0, a0;
        load(e, cr, l0, r0, a0);
        fold(e, grad(i), cr, l0, r0, a0);
    }
}

// ---------------------------------------------------------------------------
// iter_fisher with one pending gradient, float4 flavour: a thread owns four
// consecutive columns of the tile's rows, so every chain version, state array
// and new-slot store moves 16 bytes per instruction (a quarter of the memory
// instructions of the scalar kernel, the same bytes); the unit's four input
// values per sample sit in registers and the row deltas are broadcast from smem.
// Same arithmetic order per element as update_iter1_kernel.
// ---------------------------------------------------------------------------
template <int BT, int NV>
__global__ void __launch_bounds__(kThreads) update_iter1v4_kernel(const UpdArgs a) {
    FB_PDL_ENTRY();
    constexpr int RB = NV <= 6 ? 2 : 1;  // rows whose chains are loaded before any arithmetic
    __shared__ float sdel[kMaxBatch * kUpdMaxTileRows];
    const UpdWork w = a.works4[blockIdx.x];
    const int B = a.B, R = w.nrows, tid = threadIdx.x;
    const bool learn = a.eta > 0.f && a.v_r != nullptr;
    const UpdPending& pk = a.pend[0];
    auto fold1 = [&](float g, const float* cv, float& ld, float& vr, float& va) {  // one element
        float lam = a.lambda0 + ld;
        if (NV >= 2 && learn) {
            lam = iter_learn(g, cv[NV >= 2 ? 1 : 0] - cv[0], ld, vr, va, a.lambda0, a.alpha, a.eta, a.nu);
        }
        float o = g;
#pragma unroll
        for (int s = 0; s + 1 < NV; ++s) o = iter_fold(o, lam, cv[s + 1] - cv[s]);
        return sgd_new(cv[NV - 1], a.step, o);
    };
    if (w.bias) {  // one element per thread
        if (tid >= R) return;
        const int r = w.r0 + tid;
        const size_t e = (size_t)w.elem0 + r;
        float cv[NV];
#pragma unroll
        for (int i = 0; i < NV; ++i) cv[i] = __ldg(a.vers[i] + e);
        float ld = a.lam_d[e], vr = learn ? a.v_r[e] : 0.f, va = learn ? a.v_a[e] : 0.f;
        const float* dl = pk.stash + w.dlt_off + r;
        float g = 0.f;
#pragma unroll
        for (int b = 0; b < BT; ++b)
            if (b < B) g += __ldg(dl + (size_t)b * w.out);
        const float nv = fold1(g, cv, ld, vr, va);
        a.dst[e] = nv;
        if (a.dst16) reinterpret_cast<__nv_bfloat16*>(a.dst16)[e] = __float2bfloat16_rn(nv);
        if (NV >= 2 && learn) {
            a.v_r[e] = vr;
            a.v_a[e] = va;
            a.lam_d[e] = ld;
        }
        return;
    }
    const int c = w.c0 + 4 * tid;
    const bool live = c < w.in;
    float4 cv[RB][NV], st[RB][3];
    auto eoff = [&](int i) { return (size_t)w.elem0 + (size_t)(w.r0 + i) * w.in + c; };
    auto load = [&](size_t e, float4 (&v)[NV], float4 (&s3)[3]) {
#pragma unroll
        for (int k = 0; k < NV; ++k) v[k] = __ldg(reinterpret_cast<const float4*>(a.vers[k] + e));
        s3[0] = *reinterpret_cast<const float4*>(a.lam_d + e);
        s3[1] = learn ? *reinterpret_cast<const float4*>(a.v_r + e) : make_float4(0.f, 0.f, 0.f, 0.f);
        s3[2] = learn ? *reinterpret_cast<const float4*>(a.v_a + e) : make_float4(0.f, 0.f, 0.f, 0.f);
    };
#pragma unroll
    for (int i = 0; i < RB; ++i)
        if (live && i < R) load(eoff(i), cv[i], st[i]);
    for (int i = tid; i < B * R; i += blockDim.x) {
        const int b = i / R, rr = i - b * R;
        sdel[i] = __ldg(pk.stash + w.dlt_off + (size_t)b * w.out + w.r0 + rr);
    }
    float4 xv[BT];
#pragma unroll
    for (int b = 0; b < BT; ++b) {
        const float* xr = w.xin_off >= 0 ? pk.stash + w.xin_off + (size_t)b * w.in
                          : a.x0idx      ? pk.x0 + (size_t)__ldg(a.x0idx + b) * a.x0_ld
                                         : pk.x0 + (size_t)b * a.x0_ld;
        xv[b] = (b < B && live) ? __ldg(reinterpret_cast<const float4*>(xr + c)) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncthreads();
    if (!live) return;
    auto row = [&](int i, const float4 (&v)[NV], const float4 (&s3)[3]) {
        float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int b = 0; b < BT; ++b) {
            const float d = sdel[b * R + i];
            g.x = fmaf(d, xv[b].x, g.x);
            g.y = fmaf(d, xv[b].y, g.y);
            g.z = fmaf(d, xv[b].z, g.z);
            g.w = fmaf(d, xv[b].w, g.w);
        }
        float lds[4] = {s3[0].x, s3[0].y, s3[0].z, s3[0].w};
        float vrs[4] = {s3[1].x, s3[1].y, s3[1].z, s3[1].w};
        float vas[4] = {s3[2].x, s3[2].y, s3[2].z, s3[2].w};
        const float gs[4] = {g.x, g.y, g.z, g.w};
        float out[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            float cj[NV];
#pragma unroll
            for (int k = 0; k < NV; ++k) cj[k] = j == 0 ? v[k].x : j == 1 ? v[k].y : j == 2 ? v[k].z : v[k].w;
            out[j] = fold1(gs[j], cj, lds[j], vrs[j], vas[j]);
        }
        const size_t e = eoff(i);
        *reinterpret_cast<float4*>(a.dst + e) = make_float4(out[0], out[1], out[2], out[3]);
        if (a.dst16) {
            __nv_bfloat162* d16 = reinterpret_cast<__nv_bfloat162*>(reinterpret_cast<__nv_bfloat16*>(a.dst16) + e);
            d16[0] = __floats2bfloat162_rn(out[0], out[1]);
            d16[1] = __floats2bfloat162_rn(out[2], out[3]);
        }
        if (NV >= 2 && learn) {
            *reinterpret_cast<float4*>(a.lam_d + e) = make_float4(lds[0], lds[1], lds[2], lds[3]);
            *reinterpret_cast<float4*>(a.v_r + e) = make_float4(vrs[0], vrs[1], vrs[2], vrs[3]);
            *reinterpret_cast<float4*>(a.v_a + e) = make_float4(vas[0], vas[1], vas[2], vas[3]);
        }
    };
#pragma unroll
    for (int i = 0; i < RB; ++i)
        if (i < R) row(i, cv[i], st[i]);
    for (int i = RB; i < R; ++i) {
        float4 v[NV], s3[3];
        load(eoff(i), v, s3);
        row(i, v, s3);
    }
}

template <int BT>
const void* iter1v4_func(int nv) {
    switch (nv) {
#define FB_NV(n) case n: return reinterpret_cast<const void*>(&update_iter1v4_kernel<BT, n>);
        FB_NV(1) FB_NV(2) FB_NV(3) FB_NV(4) FB_NV(5) FB_NV(6) FB_NV(7) FB_NV(8)
        FB_NV(9) FB_NV(10) FB_NV(11) FB_NV(12) FB_NV(13) FB_NV(14) FB_NV(15) FB_NV(16)
#undef FB_NV
        default: return nullptr;
    }
}

// ---------------------------------------------------------------------------
// iter_fisher with one pending gradient and a chain of any length (<= 48
// versions: the deep pipelines of config 5 reach tau ~ 16-32). The version
// chain, not the arithmetic, is the cost: (nv + 3) x 4 bytes read and 16
// written per parameter. Each weight row of the tile is staged in smem with
// cp.async.bulk (one 1 KB bulk copy per version and state array, completing
// on an mbarrier), double-buffered so the copies of row i+1 are in flight
// while row i folds; the fold reads the chain from smem (consecutive threads,
// consecutive words). Bias tiles and rows that are not 16-byte aligned take
// direct loads. Arithmetic order is exactly update_iter1_kernel's.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int BT>
__global__ void __launch_bounds__(kThreads) update_stream_kernel(const UpdArgs a) {
    FB_PDL_ENTRY();
    extern __shared__ __align__(128) float sbuf[];  // 2 buffers x (nv + 3) x 256 floats
    __shared__ float sdel[kMaxBatch * kUpdMaxTileRows];
    __shared__ __align__(8) uint64_t full[2];
    const UpdTile t = a.tiles[blockIdx.x];
    const UpdSeg sg = a.segs[t.seg];
    const int B = a.B, R = t.nrows, tid = threadIdx.x, nv = a.nv;
    const bool learn = a.eta > 0.f && a.v_r != nullptr;
    const UpdPending& pk = a.pend[0];
    // fold of one element given accessors for chain version i and the state
    auto fold = [&](size_t e, float g, auto ver, float ld, float vr, float va) {
        float lam = a.lambda0 + ld;
        if (nv >= 2 && learn) {  // compensate.hpp:87-98
            lam = iter_learn(g, ver(1) - ver(0), ld, vr, va, a.lambda0, a.alpha, a.eta, a.nu);
            a.v_r[e] = vr;
            a.v_a[e] = va;
            a.lam_d[e] = ld;
        }
        float o = g;  // compensate.hpp:99-102
        float prev = ver(0);
        for (int s = 1; s < nv; ++s) {
            const float nxt = ver(s);
            o = iter_fold(o, lam, nxt - prev);
            prev = nxt;
        }
        const float nvv = sgd_new(prev, a.step, o);
        a.dst[e] = nvv;
        if (a.dst16) reinterpret_cast<__nv_bfloat16*>(a.dst16)[e] = __float2bfloat16_rn(nvv);
    };
    auto fold_global = [&](size_t e, float g) {
        fold(e, g, [&](int i) { return __ldg(a.vers[i] + e); }, a.lam_d[e], learn ? a.v_r[e] : 0.f,
             learn ? a.v_a[e] : 0.f);
    };
    if (sg.bias) {
        if (tid >= R) return;
        const int r = t.r0 + tid;
        const float* dl = pk.stash + sg.dlt_off + r;
        float g = 0.f;
#pragma unroll
        for (int b = 0; b < BT; ++b)
            if (b < B) g += __ldg(dl + (size_t)b * sg.out);
        fold_global((size_t)sg.elem0 + r, g);
        return;
    }
    for (int i = tid; i < B * R; i += kThreads) {
        const int b = i / R, rr = i - b * R;
        sdel[i] = __ldg(pk.stash + sg.dlt_off + (size_t)b * sg.out + t.r0 + rr);
    }
    const int c = t.c0 + tid;
    const int ncols = min(kUpdTileCols, sg.in - t.c0);
    float xv[BT];
#pragma unroll
    for (int b = 0; b < BT; ++b) {
        const float* xr = sg.xin_off >= 0 ? pk.stash + sg.xin_off + (size_t)b * sg.in
                          : a.x0idx       ? pk.x0 + (size_t)__ldg(a.x0idx + b) * a.x0_ld
                                          : pk.x0 + (size_t)b * a.x0_ld;
        xv[b] = (b < B && c < sg.in) ? __ldg(xr + c) : 0.f;
    }
    const bool staged = (sg.in & 3) == 0;  // 16-byte aligned rows (every version slot is 128-byte aligned)
    if (!staged) {
        __syncthreads();
        if (c >= sg.in) return;
        for (int i = 0; i < R; ++i) {
            float g = 0.f;
#pragma unroll
            for (int b = 0; b < BT; ++b) g = fmaf(sdel[b * R + i], xv[b], g);
            fold_global((size_t)sg.elem0 + (size_t)(t.r0 + i) * sg.in + c, g);
        }
        return;
    }
    const int nbuf = nv + 3;  // versions, lambda offset, v_r, v_a
    const uint32_t row_bytes = static_cast<uint32_t>(ncols) * 4u;
    auto buf = [&](int bsel, int k) { return sbuf + ((size_t)bsel * nbuf + k) * kUpdTileCols; };
    auto issue = [&](int i) {  // warp 0: bulk copies of row i into buffer i & 1
        const int bs = i & 1;
        const size_t e0 = (size_t)sg.elem0 + (size_t)(t.r0 + i) * sg.in + t.c0;
        const int ncopy = nv + (learn ? 3 : 1);
        if (tid == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&full[bs])),
                         "r"(row_bytes * ncopy)
                         : "memory");
        }
        __syncwarp();
        for (int k = tid; k < ncopy; k += 32) {
            const float* src = k < nv ? a.vers[k] + e0 : k == nv ? a.lam_d + e0 : k == nv + 1 ? a.v_r + e0 : a.v_a + e0;
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_addr(buf(bs, k))),
                "l"(src), "r"(row_bytes), "r"(smem_addr(&full[bs]))
                : "memory");
        }
    };
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&full[0])) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&full[1])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid < 32) {
        issue(0);
        if (R > 1) issue(1);
    }
    for (int i = 0; i < R; ++i) {
        const int bs = i & 1;
        {
            const uint32_t addr = smem_addr(&full[bs]), parity = (i >> 1) & 1;
            uint32_t done = 0;
            while (!done)
                asm volatile(
                    "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                    "selp.u32 %0, 1, 0, p;\n\t}"
                    : "=r"(done)
                    : "r"(addr), "r"(parity)
                    : "memory");
        }
        if (tid < ncols) {
            float g = 0.f;
#pragma unroll
            for (int b = 0; b < BT; ++b) g = fmaf(sdel[b * R + i], xv[b], g);
            const float* base = buf(bs, 0) + tid;
            fold((size_t)sg.elem0 + (size_t)(t.r0 + i) * sg.in + c, g,
                 [&](int k) { return base[(size_t)k * kUpdTileCols]; }, base[(size_t)nv * kUpdTileCols],
                 learn ? base[(size_t)(nv + 1) * kUpdTileCols] : 0.f, learn ? base[(size_t)(nv + 2) * kUpdTileCols] : 0.f);
        }
        if (i + 2 < R) {
            __syncthreads();  // every thread is done with buffer bs
            if (tid < 32) issue(i + 2);
        }
    }
}

// ---------------------------------------------------------------------------
// update_group_kernel: G <= kGroupMax consecutive iter_fisher updates of one large dense stage
// in one launch (GroupArgs, kernels.cuh): the version chain and the compensator state cross
// HBM once for the whole group instead of once per update. Persistent and warp-specialised:
// one CTA per SM walks a contiguous range of 4-row x 128-column tiles (column-block major: a
// thread keeps its column's unit inputs of all members in registers while the block lasts).
// A producer warp keeps as many tiles in flight as fit in smem (a stage: the tile's chain and
// compensator state rows, landed by 512-byte bulk copies on the stage's full barrier, plus its
// descriptor and the members' deltas of its four rows). Two consumer teams of 4 warps take
// alternate tiles, so two tiles fold at once; a thread owns one column of its tile and all
// four rows, as two f32x2 lane pairs (rows 0-1, rows 2-3): two independent dependency chains
// per thread next to the other team's. A thread forms the members' gradients, runs the
// learning steps member after member (they chain the compensator state), folds the members
// over the HBM part of the chain interleaved (segment j of the chain, between members j and
// j+1's read versions, is folded by members 0..j: one difference feeds each), hands the stage
// back (empty barrier), then member k folds the k differences its predecessors appended,
// writes version n0 + k and appends its own. Launches where a member's learning step reads an
// appended difference (it read the live version) fold member after member instead. Bias runs
// (a thread: one element) follow with direct loads. Per element the arithmetic is
// update_iter1_kernel's, update after update (bit-identical).
// ---------------------------------------------------------------------------
constexpr int kGroupChainRows = kGroupChainMax - 1;  // differences of the HBM chain (n0 <= kGroupChainMax - 1)
constexpr int kGrpMaxStages = 8;
constexpr int kGrpTeam = kGroupCols;        // consumer threads per team (a thread: one column)
constexpr int kGrpThreads = 3 * kGrpTeam;  // two consumer warpgroups + the producer warpgroup (one warp working)
constexpr size_t kGrpSmem = 212 * 1024;     // the stage ring

template <int BT>
__global__ void __launch_bounds__(kGrpThreads, 1) update_group_kernel(const __grid_constant__ GroupArgs a) {
    static_assert(kGroupRows == 4, "a consumer thread packs its four rows into two f32x2 lane pairs");
    static_assert(kGroupMax * BT <= 64, "a producer lane stages at most two deltas per tile");
    FB_PDL_ENTRY();
    extern __shared__ __align__(128) float gsm[];
    float* ring = gsm;  // [S][n_rows][4][kGroupCols]
    __shared__ float4 sdel[kGrpMaxStages][kGroupMax * BT];  // per stage: member k, sample b (rows r0 .. r0 + 3)
    __shared__ UpdWork wsm[kGrpMaxStages];
    __shared__ __align__(8) uint64_t full[kGrpMaxStages], empty[kGrpMaxStages];
    const int tid = threadIdx.x, B = a.B, G = a.G, n0 = a.n0;
    const bool learn = a.learn != 0;
    const int n_rows = n0 + (learn ? 3 : 1);  // bulk-copied rows per tile row: the chain, then the state
    constexpr int kRow = kGroupRows * kGroupCols;  // floats between a row's versions sv and sv + 1
    const size_t stage_floats = (size_t)n_rows * kRow;
    const int S = min(kGrpMaxStages, (int)(kGrpSmem / (stage_floats * sizeof(float))));
    // this CTA's contiguous range of weight tiles
    const int per = (a.n_wtiles + gridDim.x - 1) / gridDim.x;
    const int t0 = min(a.n_wtiles, (int)blockIdx.x * per), t1 = min(a.n_wtiles, t0 + per);
    if (tid == 0) {
        for (int q = 0; q < S; ++q) {
            // full: an expect_tx arrival per producer warp + one cp.async (deltas) arrival per lane of warp 0
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 36;" ::"r"(smem_addr(&full[q])) : "memory");
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(&empty[q])), "r"(kGrpTeam / 32) : "memory");
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto wait_bar = [](uint64_t* b, uint32_t parity) {
        uint32_t done = 0;
        while (!done)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                         "selp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(done)
                         : "r"(smem_addr(b)), "r"(parity)
                         : "memory");
    };
    // 12 warps = 3 per SM sub-partition at launch (<= 168 registers each); the producer
    // warpgroup hands registers to the consumer warpgroups (setmaxnreg), which need ~190
    if (tid >= 2 * kGrpTeam) {  // ---- producer warp: descriptors and deltas loaded a tile ahead
        asm volatile("setmaxnreg.dec.sync.aligned.u32 40;");
        // the warpgroup's four warps share a tile's bulk copies (each copy is issued lane after lane
        // on the uniform datapath: one warp alone cannot issue them as fast as HBM delivers); warp 0
        // also writes the descriptor and stages the deltas
        const int pw = (tid - 2 * kGrpTeam) >> 5, lane = tid & 31;
        // no global loads on this warp's path: a tile's position is decoded from the segment table
        // (kernel parameters) and its deltas land by cp.async on the stage's full barrier
        auto decode = [&](int t) {
            int s = 0;
            while (s + 1 < a.n_gsegs && t >= a.gseg[s + 1].tile0) ++s;
            const GroupSeg& gs = a.gseg[s];
            const int local = t - gs.tile0, cb = local / gs.nrt, rt = local - cb * gs.nrt;
            UpdWork w{};
            w.elem0 = gs.elem0;
            w.xin_off = gs.xin_off;
            w.dlt_off = gs.dlt_off;
            w.in = gs.in;
            w.out = gs.out;
            w.r0 = rt * kGroupRows;
            w.nrows = min(kGroupRows, gs.out - w.r0);
            w.c0 = cb * kGroupCols;
            return w;
        };
        for (int t = t0, it = 0; t < t1; ++t, ++it) {
            const int st = it % S;
            const UpdWork w = decode(t);
            if (it >= S) wait_bar(&empty[st], ((it / S) - 1) & 1);
            const int R = w.nrows, ncols = min(kGroupCols, w.in - w.c0);
            if (pw == 0 && lane == 0) wsm[st] = w;
            // deltas of member k, sample b, rows r0 .. r0 + 3 (rows past the tile's last alias it,
            // padded members / samples are zero-filled); each lane's copies arrive on full[st]
            for (int h = 0; h < 2 && pw == 0; ++h) {
                const int q = lane + 32 * h, b = q % BT, k = q / BT;
                if (q >= kGroupMax * BT) break;
                const bool ok = k < G && b < B;
                const float* dl = ok ? a.pend[k].stash + w.dlt_off + (size_t)b * w.out + w.r0 : a.vers[0];
                const uint32_t dst = smem_addr(&sdel[st][q]);
#pragma unroll
                for (int i = 0; i < kGroupRows; ++i)
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst + 4 * i), "l"(dl + (ok ? min(i, R - 1) : 0)),
                                 "r"(ok ? 4 : 0)
                                 : "memory");
            }
            if (pw == 0) asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_addr(&full[st])) : "memory");
            __syncwarp();
            const uint32_t row_bytes = static_cast<uint32_t>(ncols) * 4u;
            const int n_copy = n_rows * R;
            int mine = 0;  // copies q = pw * 32 + lane + 128 j < n_copy
            for (int q = pw * 32; q < n_copy; q += 128) mine += min(32, n_copy - q);
            // (warp 0) release: the descriptor above; every warp: the bytes of its copies
            if (lane == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&full[st])),
                             "r"(row_bytes * (uint32_t)mine)
                             : "memory");
            __syncwarp();
            float* stage = ring + st * stage_floats;
            for (int q = pw * 32 + lane; q < n_copy; q += 128) {
                const int sv = q / R, i = q - sv * R;
                const size_t off = (size_t)w.elem0 + (size_t)(w.r0 + i) * w.in + w.c0;
                const int state = sv - n0;  // >= 0: lam_d, v_r, v_a
                const float* src = state < 0 ? a.vers[sv] + off : (state == 0 ? a.lam_d : state == 1 ? a.v_r : a.v_a) + off;
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                 smem_addr(stage + (size_t)(sv * kGroupRows + i) * kGroupCols)),
                             "l"(src), "r"(row_bytes), "r"(smem_addr(&full[st]))
                             : "memory");
            }
        }
    } else {  // ---- consumer teams: team tm takes tiles it = tm, tm + 2, ...; thread lc owns column c0 + lc
        asm volatile("setmaxnreg.inc.sync.aligned.u32 232;");
        const int tm = tid / kGrpTeam, lc = tid - tm * kGrpTeam;
        // members' read versions (first chain index), uniform over the launch
        int fk[kGroupMax];
        bool interleave = true;  // read versions ascending, learning steps on HBM differences only
#pragma unroll
        for (int k = 0; k < kGroupMax; ++k) {
            fk[k] = k < G ? a.pend[k].first : n0 - 1;
            if (k < G && learn && fk[k] + 1 < n0 + k && fk[k] >= n0 - 1) interleave = false;
            if (k > 0 && k < G && fk[k] < fk[k - 1]) interleave = false;
        }
        const float lambda0 = a.lambda0, alpha = a.alpha, eta = a.eta, nu = a.nu, step = a.step;
        float xr[kGroupMax][BT];  // unit inputs x_k[b][c] of the current column block (0 past B)
        long long x_key = -1;
        const float2 lb2 = make_float2(lambda0, lambda0), oma = make_float2(__fsub_rn(1.f, alpha), __fsub_rn(1.f, alpha));
        const float2 al2 = make_float2(alpha, alpha), neta = make_float2(-eta, -eta), m2 = make_float2(-2.f, -2.f);
        const float2 nu2 = make_float2(__fmul_rn(2.f, nu), __fmul_rn(2.f, nu));
        auto sub2 = [](float2 x, float2 y) { return __fadd2_rn(x, make_float2(-y.x, -y.y)); };  // x - y, exact negation
        auto fold2 = [](float2 o, float2 lam, float2 d) { return __ffma2_rn(__fmul2_rn(__fmul2_rn(lam, o), o), d, o); };
        for (int t = t0 + tm, it = tm; t < t1; t += 2, it += 2) {
            const int st = it % S;
            wait_bar(&full[st], (it / S) & 1);
            const UpdWork w = wsm[st];
            const int R = w.nrows, c = w.c0 + lc;
            auto release = [&] {  // our smem reads ordered before the producer's next bulk copies
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if ((tid & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(&empty[st])) : "memory");
            };
            if (c >= w.in) {  // past the segment's last column: nothing to fold, hand the stage back
                release();
                continue;
            }
            const long long key = w.elem0 * 65536 + w.c0;
            if (key != x_key) {
#pragma unroll
                for (int k = 0; k < kGroupMax; ++k)
                    if (k < G) {
                        const UpdPending& pk = a.pend[k];
#pragma unroll
                        for (int b = 0; b < BT; ++b) {
                            const float* xr_p = w.xin_off >= 0 ? pk.stash + w.xin_off + (size_t)b * w.in
                                                : a.x0idx      ? pk.x0 + (size_t)__ldg(a.x0idx + b) * a.x0_ld
                                                               : pk.x0 + (size_t)b * a.x0_ld;
                            xr[k][b] = b < B ? __ldg(xr_p + c) : 0.f;
                        }
                    }
                x_key = key;
            }
            // this thread's column of the stage's four tile rows: one base, the rows at immediate
            // offsets (rows past R hold an earlier tile's values: folded, never stored)
            const float* pb = ring + st * stage_floats + lc;
            auto V = [&](int p, int sv) {
                const float* q = pb + sv * kRow + 2 * p * kGroupCols;
                return make_float2(q[0], q[kGroupCols]);
            };
            float2 ld[2], vr[2], va[2];
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                ld[p] = V(p, n0);
                vr[p] = learn ? V(p, n0 + 1) : make_float2(0.f, 0.f);
                va[p] = learn ? V(p, n0 + 2) : make_float2(0.f, 0.f);
            }
            // gradients (padded samples: delta 0 x input 0 adds +0, which leaves g unchanged)
            float2 g[kGroupMax][2];
#pragma unroll
            for (int k = 0; k < kGroupMax; ++k) {
                g[k][0] = g[k][1] = make_float2(0.f, 0.f);
                if (k < G) {
#pragma unroll
                    for (int b = 0; b < BT; ++b) {
                        const float4 dd = sdel[st][k * BT + b];
                        const float2 xx = make_float2(xr[k][b], xr[k][b]);
                        g[k][0] = __ffma2_rn(make_float2(dd.x, dd.y), xx, g[k][0]);
                        g[k][1] = __ffma2_rn(make_float2(dd.z, dd.w), xx, g[k][1]);
                    }
                }
            }
            // iter_learn in f32x2 lanes (the same rounded operations, lane by lane)
            auto learn2 = [&](int p, float2 gk, float2 d0) {
                float2 lam = __fadd2_rn(lb2, ld[p]);
                const float2 dv = __fmul2_rn(oma, sub2(gk, vr[p]));
                const float2 resid = __ffma2_rn(make_float2(-lam.x, -lam.y), va[p], dv);
                const float2 grad_l = __ffma2_rn(__fmul2_rn(m2, resid), va[p], __fmul2_rn(nu2, lam));
                ld[p] = __ffma2_rn(neta, grad_l, ld[p]);
                lam = __fadd2_rn(lb2, ld[p]);
                const float2 og = __fmul2_rn(oma, gk);
                vr[p] = __ffma2_rn(al2, vr[p], og);
                va[p] = __ffma2_rn(al2, va[p], __fmul2_rn(__fmul2_rn(og, gk), d0));
                return lam;
            };
            const size_t e0 = (size_t)w.elem0 + (size_t)w.r0 * w.in + c;
            auto store = [&](float* dk, unsigned short* dk16, int p, float2 v) {  // rows 2p, 2p + 1 if inside the tile
                const size_t ea = e0 + (size_t)(2 * p) * w.in, eb = ea + (size_t)w.in;
                if (2 * p < R) {
                    dk[ea] = v.x;
                    if (dk16) reinterpret_cast<__nv_bfloat16*>(dk16)[ea] = __float2bfloat16_rn(v.x);
                }
                if (2 * p + 1 < R) {
                    dk[eb] = v.y;
                    if (dk16) reinterpret_cast<__nv_bfloat16*>(dk16)[eb] = __float2bfloat16_rn(v.y);
                }
            };
            float2 dt[kGroupMax][2];  // differences appended by the members
            float2 cur[2];
            if (interleave) {
                float2 lam[kGroupMax][2], o[kGroupMax][2];
#pragma unroll
                for (int k = 0; k < kGroupMax; ++k)
#pragma unroll
                    for (int p = 0; p < 2; ++p) {
                        o[k][p] = g[k][p];
                        lam[k][p] = __fadd2_rn(lb2, ld[p]);
                        if (k < G && learn && fk[k] + 1 < n0 + k) lam[k][p] = learn2(p, g[k][p], sub2(V(p, fk[k] + 1), V(p, fk[k])));
                    }
                // the HBM chain's differences in one ascending pass: segment j, [fk[j], fk[j + 1]),
                // is folded by members 0..j
                float2 vp[2] = {V(0, fk[0]), V(1, fk[0])};
#pragma unroll
                for (int j = 0; j < kGroupMax; ++j)
                    if (j < G) {
                        const int hi = j + 1 < G ? fk[j + 1] : n0 - 1;
                        for (int sv = fk[j]; sv < hi; ++sv) {
#pragma unroll
                            for (int p = 0; p < 2; ++p) {
                                const float2 vn = V(p, sv + 1);
                                const float2 d = sub2(vn, vp[p]);
                                vp[p] = vn;
#pragma unroll
                                for (int m = 0; m <= j; ++m) o[m][p] = fold2(o[m][p], lam[m][p], d);
                            }
                        }
                    }
                release();
                cur[0] = vp[0];  // version n0 - 1
                cur[1] = vp[1];
#pragma unroll
                for (int k = 0; k < kGroupMax; ++k)
                    if (k < G)
#pragma unroll
                        for (int p = 0; p < 2; ++p) {
                            float2 ok = o[k][p];
#pragma unroll
                            for (int j = 0; j < k; ++j) ok = fold2(ok, lam[k][p], dt[j][p]);
                            const float2 nv = make_float2(sgd_new(cur[p].x, step, ok.x), sgd_new(cur[p].y, step, ok.y));
                            dt[k][p] = sub2(nv, cur[p]);
                            cur[p] = nv;
                            store(a.dst[k], a.dst16[k], p, nv);
                        }
            } else {
                cur[0] = V(0, n0 - 1);
                cur[1] = V(1, n0 - 1);
#pragma unroll
                for (int k = 0; k < kGroupMax; ++k)
                    if (k < G) {
                        const int first = fk[k];
#pragma unroll
                        for (int p = 0; p < 2; ++p) {
                            float2 lam = __fadd2_rn(lb2, ld[p]);
                            if (learn && first + 1 < n0 + k) {
                                float2 d0 = first < n0 - 1 ? sub2(V(p, first + 1), V(p, first)) : dt[0][p];
#pragma unroll
                                for (int j = 1; j < k; ++j)
                                    if (first == n0 - 1 + j) d0 = dt[j][p];
                                lam = learn2(p, g[k][p], d0);
                            }
                            float2 o = g[k][p];
                            if (first + 1 < n0) {
                                float2 vp = V(p, first);
                                for (int sv = first; sv + 1 < n0; ++sv) {
                                    const float2 vn = V(p, sv + 1);
                                    o = fold2(o, lam, sub2(vn, vp));
                                    vp = vn;
                                }
                            }
#pragma unroll
                            for (int j = 0; j < k; ++j)
                                if (n0 - 1 + j >= first) o = fold2(o, lam, dt[j][p]);
                            const float2 nv = make_float2(sgd_new(cur[p].x, step, o.x), sgd_new(cur[p].y, step, o.y));
                            dt[k][p] = sub2(nv, cur[p]);
                            cur[p] = nv;
                            store(a.dst[k], a.dst16[k], p, nv);
                        }
                    }
                release();
            }
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                store(a.lam_d, nullptr, p, ld[p]);
                if (learn) {
                    store(a.v_r, nullptr, p, vr[p]);
                    store(a.v_a, nullptr, p, va[p]);
                }
            }
        }
    }
    // bias runs (after the weight tiles): a thread per element, direct loads
    for (int t = a.n_wtiles + blockIdx.x; t < a.n_tiles; t += gridDim.x) {
        const UpdWork w = a.works[t];
        if (tid >= w.nrows || tid >= 2 * kGrpTeam) continue;
        const size_t e = (size_t)w.elem0 + w.r0 + tid;
        float prev = __ldg(a.vers[0] + e);
        float d[kGroupChainRows];
        int n = a.n0;
        for (int sv = 0; sv + 1 < n; ++sv) {
            const float nxt = __ldg(a.vers[sv + 1] + e);
            d[sv] = nxt - prev;
            prev = nxt;
        }
        float cur = prev, ld = a.lam_d[e], vr = learn ? a.v_r[e] : 0.f, va = learn ? a.v_a[e] : 0.f;
        for (int k = 0; k < G; ++k) {
            const UpdPending& pk = a.pend[k];
            const int first = pk.first;
            float g = 0.f;
            const float* dl = pk.stash + w.dlt_off + w.r0 + tid;
            for (int b = 0; b < BT; ++b)
                if (b < B) g += __ldg(dl + (size_t)b * w.out);
            float lam = a.lambda0 + ld;
            if (learn && first + 1 < n) lam = iter_learn(g, d[first], ld, vr, va, a.lambda0, a.alpha, a.eta, a.nu);
            float o = g;
            for (int sv = first; sv + 1 < n; ++sv) o = iter_fold(o, lam, d[sv]);
            const float nv = sgd_new(cur, a.step, o);
            d[n - 1] = nv - cur;
            cur = nv;
            a.dst[k][e] = nv;
            if (a.dst16[k]) reinterpret_cast<__nv_bfloat16*>(a.dst16[k])[e] = __float2bfloat16_rn(nv);
            ++n;
        }
        a.lam_d[e] = ld;
        if (learn) {
            a.v_r[e] = vr;
            a.v_a[e] = va;
        }
    }
}

template <int BT>
const void* group_func() {
    static const void* f = [] {
        const void* p = reinterpret_cast<const void*>(&update_group_kernel<BT>);
        cudaFuncSetAttribute(p, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGrpSmem);
        return p;
    }();
    return f;
}

template <int BT>
const void* stream_func(size_t smem) {
    static size_t configured = 0;  // (static smem counts against the 48 KB default too)
    const void* f = reinterpret_cast<const void*>(&update_stream_kernel<BT>);
    if (smem > configured) {
        cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured = smem;
    }
    return f;
}

template <int BT>
const void* iter1_func(int nv) {
    switch (nv) {
#define FB_NV(n) case n: return reinterpret_cast<const void*>(&update_iter1_kernel<BT, n>);
        FB_NV(1) FB_NV(2) FB_NV(3) FB_NV(4) FB_NV(5) FB_NV(6) FB_NV(7) FB_NV(8)
        FB_NV(9) FB_NV(10) FB_NV(11) FB_NV(12) FB_NV(13) FB_NV(14) FB_NV(15) FB_NV(16)
#undef FB_NV
        default: return nullptr;
    }
}

template <int POLICY>
const void* update_func(int B) {
    if (B <= 1) return reinterpret_cast<const void*>(&update_tile_kernel<POLICY, 1>);
    if (B <= 2) return reinterpret_cast<const void*>(&update_tile_kernel<POLICY, 2>);
    if (B <= 4) return reinterpret_cast<const void*>(&update_tile_kernel<POLICY, 4>);
    if (B <= 8) return reinterpret_cast<const void*>(&update_tile_kernel<POLICY, 8>);
    return reinterpret_cast<const void*>(&update_tile_kernel<POLICY, 16>);
}

// ---------------------------------------------------------------------------
// unit compensation kernel (flat, absolute lambda)
// ---------------------------------------------------------------------------
template <int POLICY>
__global__ void __launch_bounds__(kThreads) compensate_kernel(const CompArgs a) {
    FB_PDL_ENTRY();
    const long long stride = (long long)gridDim.x * blockDim.x;
    const bool learn = a.eta > 0.f && a.v_r != nullptr;
    const int last = a.chain_len - 1;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < a.n; e += stride) {
        ElemState st{0.f, 0.f, 0.f, 0.f};
        if (POLICY == 4) {
            st.ld = a.lambda[e];
            if (learn) { st.vr = a.v_r[e]; st.va = a.v_a[e]; }
        }
        if (POLICY == 2) st.gp = a.gap[e];
        const float thc = a.chain[last][e];
        a.out[e] = compensate_elem<POLICY>(a.g[e], a.chain, 0, last, (size_t)e, thc, st,
                                           POLICY == 4 ? 0.f : a.lambda0, a.alpha, a.eta, a.nu, learn);
        if (POLICY == 4) {
            a.lambda[e] = st.ld;
            if (learn) { a.v_r[e] = st.vr; a.v_a[e] = st.va; }
        }
        if (POLICY == 2) a.gap[e] = st.gp;
    }
}

// ---------------------------------------------------------------------------
// RunningNormalizer: thread per feature, items in arrival order. The explicit
// _rn intrinsics forbid FMA contraction so the result matches the host's
// separately rounded multiply/add (x86-64 SSE2, no FMA) bit for bit.
// ---------------------------------------------------------------------------
__global__ void normalize_kernel(const NormArgs a) {
    FB_PDL_ENTRY();
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= a.F) return;
    double mu = a.mean[f], m2 = a.m2[f];
    unsigned long long cnt = *a.count_base + a.count_off;
    for (long long i = 0; i < a.n; ++i) {
        const double x = a.raw[i * a.F + f];
        if (!a.apply_only) {
            ++cnt;
            const double d = __dsub_rn(x, mu);
            mu = __dadd_rn(mu, __ddiv_rn(d, (double)cnt));
            m2 = __dadd_rn(m2, __dmul_rn(d, __dsub_rn(x, mu)));
        }
        const double var = cnt > 1 ? __ddiv_rn(m2, (double)(cnt - 1)) : 1.0;
        const double sd = __dsqrt_rn(var < 1e-8 ? 1e-8 : var);
        a.out[i * a.F + f] = (float)__ddiv_rn(__dsub_rn(x, mu), sd);
    }
    if (!a.apply_only) {
        a.mean[f] = mu;
        a.m2[f] = m2;
    }
}

// Two-phase RunningNormalizer (same arithmetic, same bits as normalize_kernel).
// Only mean and M2 form a recurrence over the samples; the standardisation of
// sample i (variance, sqrt, divide: most of the fp64 latency) depends on
// (mean_i, M2_i) alone. Phase 1 walks the recurrence per feature and records
// (mean_i, M2_i); phase 2 standardises every (sample, feature) in parallel.
__global__ void welford_kernel(const NormArgs a) {
    FB_PDL_ENTRY();
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= a.F) return;
    double mu = a.mean[f], m2 = a.m2[f];
    unsigned long long cnt = *a.count_base + a.count_off;
#pragma unroll 4
    for (long long i = 0; i < a.n; ++i) {
        const double x = a.raw[i * a.F + f];
        ++cnt;
        const double d = __dsub_rn(x, mu);
        mu = __dadd_rn(mu, __ddiv_rn(d, (double)cnt));
        m2 = __dadd_rn(m2, __dmul_rn(d, __dsub_rn(x, mu)));
        a.mu_i[i * a.F + f] = mu;
        a.m2_i[i * a.F + f] = m2;
    }
    a.mean[f] = mu;
    a.m2[f] = m2;
}

__global__ void standardize_kernel(const NormArgs a) {
    FB_PDL_ENTRY();
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= a.n * a.F) return;
    const long long i = t / a.F;
    const unsigned long long cnt = *a.count_base + a.count_off + (unsigned long long)i + 1;
    const double x = a.raw[t], mu = a.mu_i[t], m2 = a.m2_i[t];
    const double var = cnt > 1 ? __ddiv_rn(m2, (double)(cnt - 1)) : 1.0;
    const double sd = __dsqrt_rn(var < 1e-8 ? 1e-8 : var);
    a.out[t] = (float)__ddiv_rn(__dsub_rn(x, mu), sd);
}

// Replay-pool insertion: one CTA per sample of the unit.
__global__ void pool_kernel(const PoolArgs a) {
    FB_PDL_ENTRY();
    const int b = blockIdx.x;
    const int dst = a.dst[b];
    if (dst < 0) return;
    const float* src = a.x + (size_t)b * a.F;
    float* out = a.pool_x + (size_t)dst * a.F;
    for (int f = threadIdx.x; f < a.F; f += blockDim.x) out[f] = src[f];
    if (threadIdx.x == 0) a.pool_labels[dst] = a.labels[b];
}

// Hand-off between ranks. One CTA each: messages are B x width floats (<= 256 KB).
// Flow control without host barriers: a message slot of chunk e may be overwritten
// only once its receiver consumed it in chunk e - 1, which the receiver reports by
// storing e - 1 into the sender's ack slot (recv_kernel); the sender waits for it.
__device__ __forceinline__ bool wait_epoch(const unsigned* word, unsigned want, bool exact, unsigned* error) {
    unsigned v;
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(word) : "memory");
        if (exact ? v == want : static_cast<int>(v - want) >= 0) return true;
        __nanosleep(64);
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > 10000000000ull) {  // a peer rank is not progressing: fail the chunk, never hang
            if (error) atomicExch(error, 1u);
            return false;
        }
    }
}

__global__ void __launch_bounds__(512) send_kernel(const SendArgs a) {
    FB_PDL_ENTRY();
    if (a.ack) {
        __shared__ unsigned go;
        if (threadIdx.x == 0) go = wait_epoch(a.ack, *a.epoch - 1u, false, a.error);
        __syncthreads();
        (void)go;
    }
    const bool vec = ((reinterpret_cast<uintptr_t>(a.src) | reinterpret_cast<uintptr_t>(a.dst)) & 15u) == 0 && (a.n & 3) == 0;
    if (vec) {
        const float4* s = reinterpret_cast<const float4*>(a.src);
        float4* d = reinterpret_cast<float4*>(a.dst);
        for (int i = threadIdx.x; i < a.n / 4; i += blockDim.x) d[i] = s[i];
    } else {
        for (int i = threadIdx.x; i < a.n; i += blockDim.x) a.dst[i] = a.src[i];
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned e = *a.epoch;
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(a.flag), "r"(e) : "memory");
    }
}

__global__ void __launch_bounds__(512) recv_kernel(const RecvArgs a) {
    FB_PDL_ENTRY();
    __shared__ unsigned ready;
    const unsigned e = *a.epoch;
    if (threadIdx.x == 0) ready = wait_epoch(a.flag, e, true, a.error);
    __syncthreads();
    (void)ready;
    for (int i = threadIdx.x; i < a.n; i += blockDim.x) {
        float v = __ldcv(a.src + i);  // bypass L1: the peer wrote it
        if (a.mask && !(a.mask[i] > 0.f)) v = 0.f;
        a.dst[i] = v;
    }
    if (a.ack) {  // every read of the slot is done: the sender may reuse it next chunk
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence_system();
            asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(a.ack), "r"(e) : "memory");
        }
    }
}

} // namespace

void spec_send(const SendArgs& a, KernelSpec& k) {
    fill(k, reinterpret_cast<const void*>(&send_kernel), dim3(1), dim3(512), a);
}

void spec_recv(const RecvArgs& a, KernelSpec& k) {
    fill(k, reinterpret_cast<const void*>(&recv_kernel), dim3(1), dim3(512), a);
}

void spec_fwd(const FwdArgs& a, KernelSpec& k) {
    // rows are b * in (or xidx[b] * in) floats from X: float4 needs in % 4 == 0 and aligned bases
    const bool vec = (a.in & 3) == 0 && aligned16(a.W) && aligned16(a.X);
    if (a.B <= 1) fwd_spec<1, 4>(a, vec, k);
    else if (a.B <= 2) fwd_spec<2, 4>(a, vec, k);
    else if (a.B <= 4) fwd_spec<4, 4>(a, vec, k);
    else if (a.B <= 8) fwd_spec<8, 4>(a, vec, k);
    else fwd_spec<16, 2>(a, vec, k);
}

bool fwd_single_cta(int in, int out, int B, bool vec) {
    const int RW = B <= 8 ? 4 : 2;  // spec_fwd's choice
    return out <= fwd_rows_per_cta(in, vec, RW);
}

void spec_head(const HeadArgs& a, KernelSpec& k) {
    fill(k, reinterpret_cast<const void*>(&head_kernel), dim3((a.B + kWarps - 1) / kWarps), dim3(kThreads), a);
}

static int bwd_vec(int in) { return (in & 3) == 0 ? 4 : 1; }

int bwd_col_tiles(int in) {
    const int tc = 32 * bwd_vec(in);
    return (in + tc - 1) / tc;
}

int bwd_row_splits(int in, int out) {
    const int tiles = bwd_col_tiles(in);
    int splits = (2 * 148 + tiles - 1) / tiles;
    const int max_by_rows = (out + 31) / 32;  // >= 4 rows per warp (one unrolled trip)
    if (splits > max_by_rows) splits = max_by_rows;
    const int min_for_smem = (out + kBwdMaxRows - 1) / kBwdMaxRows;
    if (splits < min_for_smem) splits = min_for_smem;
    return splits < 1 ? 1 : splits;
}

template <int BT, int V>
static const void* bwd_func_v(size_t& smem) {
    smem = sizeof(float) * kWarps * BT * 32 * V;
    static bool configured = false;  // > 48 KB dynamic smem needs an opt-in per function
    if (!configured) {
        cudaFuncSetAttribute(reinterpret_cast<const void*>(&bwd_kernel<BT, V>), cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        configured = true;
    }
    return reinterpret_cast<const void*>(&bwd_kernel<BT, V>);
}

template <int BT>
static const void* bwd_func(bool vec, size_t& smem) {
    return vec ? bwd_func_v<BT, 4>(smem) : bwd_func_v<BT, 1>(smem);
}

void spec_bwd(const BwdArgs& a, KernelSpec& k) {
    if (a.out <= kBwdSmallRows) {
        const void* f = a.B <= 1 ? reinterpret_cast<const void*>(&bwd_small_kernel<1>)
                      : a.B <= 2 ? reinterpret_cast<const void*>(&bwd_small_kernel<2>)
                      : a.B <= 4 ? reinterpret_cast<const void*>(&bwd_small_kernel<4>)
                      : a.B <= 8 ? reinterpret_cast<const void*>(&bwd_small_kernel<8>)
                                 : reinterpret_cast<const void*>(&bwd_small_kernel<16>);
        fill(k, f, dim3((a.in + 31) / 32), dim3(kThreads), a);
        return;
    }
    const dim3 grid(bwd_col_tiles(a.in), a.row_splits);
    const bool vec = bwd_vec(a.in) == 4 && aligned16(a.W);
    size_t smem = 0;
    const void* f = a.B <= 1 ? bwd_func<1>(vec, smem) : a.B <= 2 ? bwd_func<2>(vec, smem) : a.B <= 4 ? bwd_func<4>(vec, smem)
                  : a.B <= 8 ? bwd_func<8>(vec, smem) : bwd_func<16>(vec, smem);
    fill(k, f, grid, dim3(kThreads), a);
    k.smem = smem;
}

void spec_update(const UpdArgs& a, KernelSpec& k) {
    const long long blocks = a.n_tiles;
    // FERRET_STREAM_MIN_CHAIN (test / experiment knob): chain length above which
    // the smem-staged kernel takes over from the register-resident one
    if (a.gmat && !(a.policy == 4 && a.K == 1 && a.nv <= 16 && a.lam_d != nullptr)) {
        // materialised gradients (conv stages) outside the iter1 kernel's case: the generic tile kernel
        const void* f = a.policy == 0 ? update_func<0>(a.B) : a.policy == 1 ? update_func<1>(a.B)
                      : a.policy == 2 ? update_func<2>(a.B) : a.policy == 3 ? update_func<3>(a.B) : update_func<4>(a.B);
        fill(k, f, dim3((unsigned)blocks), dim3(kThreads), a);
        return;
    }
    // Stages of >= 8 M parameters (chains of 32 MB versions, far beyond L2) stream every chain
    // longer than 4 versions through smem: C5 fp32 3.51k -> 3.74k samples/s against the
    // register-resident kernel up to 16 (profiles/r2/stream_chain_ab.txt); small L2-resident
    // stages keep the latency-shaped register kernel up to 16 versions
    const char* env = std::getenv("FERRET_STREAM_MIN_CHAIN");
    const int min_chain = env ? std::atoi(env) : a.n_elems >= (8ll << 20) ? kStreamMinChainLarge : kStreamMinChain;
    if (!a.gmat && a.policy == 4 && a.K == 1 && a.nv > min_chain && a.lam_d != nullptr) {
        const size_t smem = sizeof(float) * 2 * (size_t)(a.nv + 3) * kUpdTileCols;
        const void* f = a.B <= 1 ? stream_func<1>(smem) : a.B <= 2 ? stream_func<2>(smem) : a.B <= 4 ? stream_func<4>(smem)
                      : a.B <= 8 ? stream_func<8>(smem) : stream_func<16>(smem);
        fill(k, f, dim3((unsigned)blocks), dim3(kThreads), a);
        k.smem = smem;
        return;
    }
    // FERRET_UPDATE_V4=0 (experiment knob) keeps the scalar kernel
    static const bool v4_on = !std::getenv("FERRET_UPDATE_V4") || std::atoi(std::getenv("FERRET_UPDATE_V4")) != 0;
    if (v4_on && !a.gmat && a.policy == 4 && a.K == 1 && a.nv <= 16 && a.lam_d != nullptr && a.works4 != nullptr) {
        const void* f = a.B <= 1 ? iter1v4_func<1>(a.nv) : a.B <= 2 ? iter1v4_func<2>(a.nv) : a.B <= 4 ? iter1v4_func<4>(a.nv)
                      : a.B <= 8 ? iter1v4_func<8>(a.nv) : iter1v4_func<16>(a.nv);
        fill(k, f, dim3((unsigned)a.n_tiles4), dim3(a.threads4), a);
        return;
    }
    if (a.policy == 4 && a.K == 1 && a.nv <= 16 && a.lam_d != nullptr) {
        static const bool pipe = !std::getenv("FERRET_UPDATE_PIPELINE") || std::atoi(std::getenv("FERRET_UPDATE_PIPELINE")) != 0;
        UpdArgs b = a;
        b.pipe = pipe ? 1 : 0;
        const void* f = a.B <= 1 ? iter1_func<1>(a.nv) : a.B <= 2 ? iter1_func<2>(a.nv) : a.B <= 4 ? iter1_func<4>(a.nv)
                      : a.B <= 8 ? iter1_func<8>(a.nv) : iter1_func<16>(a.nv);
        fill(k, f, dim3((unsigned)blocks), dim3(kThreads), b);
        k.chain_pdl = true;
        return;
    }
    const void* f = a.policy == 0 ? update_func<0>(a.B) : a.policy == 1 ? update_func<1>(a.B)
                  : a.policy == 2 ? update_func<2>(a.B) : a.policy == 3 ? update_func<3>(a.B) : update_func<4>(a.B);
    fill(k, f, dim3((unsigned)blocks), dim3(kThreads), a);
}

void spec_update_group(const GroupArgs& a, KernelSpec& k) {
    const void* f = a.B <= 1 ? group_func<1>() : a.B <= 2 ? group_func<2>() : a.B <= 4 ? group_func<4>()
                  : a.B <= 8 ? group_func<8>() : group_func<16>();
    // persistent: one CTA per SM (at most one per tile)
    fill(k, f, dim3((unsigned)std::max(1, std::min(a.n_tiles, 148))), dim3(kGrpThreads), a);
    k.smem = kGrpSmem;
}

void spec_normalize(const NormArgs& a, KernelSpec& k) {
    fill(k, reinterpret_cast<const void*>(&normalize_kernel), dim3((a.F + 127) / 128), dim3(128), a);
}

void spec_welford(const NormArgs& a, KernelSpec& k) {
    fill(k, reinterpret_cast<const void*>(&welford_kernel), dim3((a.F + 63) / 64), dim3(64), a);
}

void spec_standardize(const NormArgs& a, KernelSpec& k) {
    const long long n = a.n * a.F;
    fill(k, reinterpret_cast<const void*>(&standardize_kernel), dim3((unsigned)((n + 255) / 256)), dim3(256), a);
}

void spec_pool(const PoolArgs& a, KernelSpec& k) {
    fill(k, reinterpret_cast<const void*>(&pool_kernel), dim3(a.B), dim3(128), a);
}

cudaError_t launch_spec(KernelSpec& k, cudaStream_t s) {
    return cudaLaunchKernel(k.func, k.grid, k.block, k.kernel_params(), k.smem, s);
}

void launch_compensate(const CompArgs& a, cudaStream_t s) {
    long long blocks = (a.n + kThreads - 1) / kThreads;
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks < 1) blocks = 1;
    switch (a.policy) {
        case 0: compensate_kernel<0><<<(int)blocks, kThreads, 0, s>>>(a); break;
        case 1: compensate_kernel<1><<<(int)blocks, kThreads, 0, s>>>(a); break;
        case 2: compensate_kernel<2><<<(int)blocks, kThreads, 0, s>>>(a); break;
        case 3: compensate_kernel<3><<<(int)blocks, kThreads, 0, s>>>(a); break;
        default: compensate_kernel<4><<<(int)blocks, kThreads, 0, s>>>(a); break;
    }
}

} // namespace fb200
