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

#include <cfloat>
#include <cstdio>

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

// ---------------------------------------------------------------------------
// forward: warp per RW output rows; lanes stream the weight rows with float4
// loads; each weight load is reused by the B samples (registers) and each
// input load by the RW rows.
// ---------------------------------------------------------------------------
template <int BT, int RW, bool VEC>
__global__ void __launch_bounds__(kThreads) fwd_kernel(const FwdArgs a) {
    const int lane = threadIdx.x & 31;
    const int gwarp = blockIdx.x * kWarps + (threadIdx.x >> 5);
    const int nwarps = gridDim.x * kWarps;
    const int B = a.B;
    for (int r0 = gwarp * RW; r0 < a.out; r0 += nwarps * RW) {
        float acc[RW][BT];
#pragma unroll
        for (int i = 0; i < RW; ++i)
#pragma unroll
            for (int b = 0; b < BT; ++b) acc[i][b] = 0.f;
        if (VEC) {
            const int n4 = a.in >> 2;
            for (int c4 = lane; c4 < n4; c4 += 32) {
                float4 xv[BT];
#pragma unroll
                for (int b = 0; b < BT; ++b)
                    xv[b] = b < B ? __ldg(reinterpret_cast<const float4*>(a.X + a.xoff[b]) + c4)
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int i = 0; i < RW; ++i) {
                    const int r = r0 + i;
                    if (r >= a.out) break;
                    const float4 w = __ldg(reinterpret_cast<const float4*>(a.W + (size_t)r * a.in) + c4);
#pragma unroll
                    for (int b = 0; b < BT; ++b) {
                        acc[i][b] = fmaf(w.x, xv[b].x, acc[i][b]);
                        acc[i][b] = fmaf(w.y, xv[b].y, acc[i][b]);
                        acc[i][b] = fmaf(w.z, xv[b].z, acc[i][b]);
                        acc[i][b] = fmaf(w.w, xv[b].w, acc[i][b]);
                    }
                }
            }
        } else {
            for (int c = lane; c < a.in; c += 32) {
                float xv[BT];
#pragma unroll
                for (int b = 0; b < BT; ++b) xv[b] = b < B ? __ldg(a.X + a.xoff[b] + c) : 0.f;
#pragma unroll
                for (int i = 0; i < RW; ++i) {
                    const int r = r0 + i;
                    if (r >= a.out) break;
                    const float w = __ldg(a.W + (size_t)r * a.in + c);
#pragma unroll
                    for (int b = 0; b < BT; ++b) acc[i][b] = fmaf(w, xv[b], acc[i][b]);
                }
            }
        }
#pragma unroll
        for (int i = 0; i < RW; ++i) {
            const int r = r0 + i;
#pragma unroll
            for (int b = 0; b < BT; ++b) {
                const float s = warp_sum(acc[i][b]);
                if (lane == b && b < B && r < a.out) {
                    float z = s + a.bias[r];
                    if (a.relu) z = z > 0.f ? z : 0.f;
                    a.Y[(size_t)b * a.out + r] = z;
                }
            }
        }
    }
}

template <int BT, int RW>
void fwd_dispatch_vec(const FwdArgs& a, cudaStream_t s, bool vec) {
    const int rows_per_cta = kWarps * RW;
    int grid = (a.out + rows_per_cta - 1) / rows_per_cta;
    if (grid > 148 * 16) grid = 148 * 16;
    if (vec) fwd_kernel<BT, RW, true><<<grid, kThreads, 0, s>>>(a);
    else fwd_kernel<BT, RW, false><<<grid, kThreads, 0, s>>>(a);
}

// ---------------------------------------------------------------------------
// softmax head: one warp per sample.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) head_kernel(const HeadArgs a) {
    const int lane = threadIdx.x & 31;
    const int b = blockIdx.x * kWarps + (threadIdx.x >> 5);
    if (b >= a.B) return;
    const float* z = a.logits + (size_t)b * a.n_out;
    // max with first-index tie break
    float best = -FLT_MAX;
    int best_k = 0x7fffffff;
    for (int k = lane; k < a.n_out; k += 32) {
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
    if (a.mode == 0) {
        if (lane == 0) a.pred[b] = best_k;
        return;
    }
    float sum = 0.f;
    for (int k = lane; k < a.n_out; k += 32) sum += expf(z[k] - best);
    sum = warp_sum(sum);
    const int label = a.labels[b];
    float* d = a.delta + (size_t)b * a.n_out;
    for (int k = lane; k < a.n_out; k += 32) {
        const float p = expf(z[k] - best) / sum;
        d[k] = a.scale * (k == label ? p - 1.f : p);
    }
}

// ---------------------------------------------------------------------------
// backward delta propagation: thread per input column; the output rows are
// split over grid.y and the last CTA of a column tile reduces the partial sums
// in split order (deterministic).
// ---------------------------------------------------------------------------
constexpr int kBwdCols = 256;
constexpr int kBwdMaxRowsPerSplit = 256;

template <int BT>
__global__ void __launch_bounds__(kBwdCols) bwd_kernel(const BwdArgs a) {
    __shared__ float sd[BT][kBwdMaxRowsPerSplit];
    __shared__ bool last_cta;
    const int c = blockIdx.x * kBwdCols + threadIdx.x;
    const int splits = gridDim.y;
    const int rows_per = (a.out + splits - 1) / splits;
    const int r_begin = blockIdx.y * rows_per;
    const int r_end = min(a.out, r_begin + rows_per);
    const int B = a.B;
    for (int i = threadIdx.x; i < BT * rows_per; i += kBwdCols) {
        const int b = i / rows_per, rr = i % rows_per;
        const int r = r_begin + rr;
        sd[b][rr] = (b < B && r < r_end) ? a.d_out[(size_t)b * a.out + r] : 0.f;
    }
    __syncthreads();
    float acc[BT];
#pragma unroll
    for (int b = 0; b < BT; ++b) acc[b] = 0.f;
    if (c < a.in) {
        const float* w = a.W + (size_t)r_begin * a.in + c;
        int r = r_begin;
        for (; r + 4 <= r_end; r += 4) {
            const float w0 = __ldg(w), w1 = __ldg(w + a.in), w2 = __ldg(w + 2 * (size_t)a.in),
                        w3 = __ldg(w + 3 * (size_t)a.in);
            w += 4 * (size_t)a.in;
            const int rr = r - r_begin;
#pragma unroll
            for (int b = 0; b < BT; ++b) {
                acc[b] = fmaf(w0, sd[b][rr], acc[b]);
                acc[b] = fmaf(w1, sd[b][rr + 1], acc[b]);
                acc[b] = fmaf(w2, sd[b][rr + 2], acc[b]);
                acc[b] = fmaf(w3, sd[b][rr + 3], acc[b]);
            }
        }
        for (; r < r_end; ++r) {
            const float w0 = __ldg(w);
            w += a.in;
#pragma unroll
            for (int b = 0; b < BT; ++b) acc[b] = fmaf(w0, sd[b][r - r_begin], acc[b]);
        }
    }
    if (splits == 1) {
        if (c < a.in) {
#pragma unroll
            for (int b = 0; b < BT; ++b) {
                if (b >= B) break;
                float v = acc[b];
                if (a.mask && !(a.mask[(size_t)b * a.in + c] > 0.f)) v = 0.f;
                a.d_in[(size_t)b * a.in + c] = v;
            }
        }
        return;
    }
    if (c < a.in) {
#pragma unroll
        for (int b = 0; b < BT; ++b)
            if (b < B) a.partial[((size_t)blockIdx.y * B + b) * a.in + c] = acc[b];
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned ticket = atomicAdd(&a.counters[blockIdx.x], 1u);
        last_cta = ticket == (unsigned)(splits - 1);
    }
    __syncthreads();
    if (!last_cta) return;
    __threadfence();
    if (c < a.in) {
        for (int b = 0; b < B; ++b) {
            float v = 0.f;
            for (int sp = 0; sp < splits; ++sp) v += __ldcg(a.partial + ((size_t)sp * B + b) * a.in + c);
            if (a.mask && !(a.mask[(size_t)b * a.in + c] > 0.f)) v = 0.f;
            a.d_in[(size_t)b * a.in + c] = v;
        }
    }
    if (threadIdx.x == 0) a.counters[blockIdx.x] = 0u;
}

// ---------------------------------------------------------------------------
// compensation of one element for one pending gradient (compensate.hpp).
// `ver(v)` returns the base pointer of parameter version v; the chain is
// versions first_v .. cur_v (cur_v's value at element e is th_cur).
// ---------------------------------------------------------------------------
struct ElemState {
    float ld, vr, va, gp;
};

struct RingVersions {
    const float* ring;
    long long slot_floats;
    int depth;
    __device__ __forceinline__ const float* operator()(long long v) const {
        return ring + (v % depth) * slot_floats;
    }
};

struct ListVersions {
    const float* const* p;
    __device__ __forceinline__ const float* operator()(long long v) const { return p[v]; }
};

template <int POLICY, class Ver>
__device__ __forceinline__ float compensate_elem(float g, const Ver& ver, long long first_v, long long cur_v,
                                                 size_t e, float th_cur, ElemState& st, float lam_base,
                                                 float alpha, float eta, float nu, bool learn) {
    const long long tau = cur_v - first_v;
    if (POLICY == 0) {  // none
        return g;
    } else if (POLICY == 1) {  // step: g * 1/(1+tau)              compensate.hpp:107-113
        return g * (1.f / (1.f + (float)tau));
    } else if (POLICY == 2) {  // gap                               compensate.hpp:117-130, learner.hpp:104-111
        const float read = __ldg(ver(first_v) + e);
        const float gapv = fabsf(th_cur - read);
        const float mg = fmaxf(st.gp, 1e-12f);
        const float o = g / (1.f + gapv / mg);
        st.gp = 0.99f * st.gp + 0.01f * gapv;
        return o;
    } else if (POLICY == 3) {  // fisher: g + lambda0 g^2 (cur - read)   compensate.hpp:42-51
        const float read = __ldg(ver(first_v) + e);
        return g + lam_base * g * g * (th_cur - read);
    } else {  // iter_fisher                                            compensate.hpp:82-104
        float lam = lam_base + st.ld;
        float prev = tau >= 1 ? __ldg(ver(first_v) + e) : th_cur;
        if (learn && tau >= 1) {
            const float one_m_a = 1.f - alpha;
            const float dv = one_m_a * (g - st.vr);
            const float resid = dv - lam * st.va;
            const float grad_l = -2.f * resid * st.va + 2.f * nu * lam;
            st.ld -= eta * grad_l;
            lam = lam_base + st.ld;
            const float nxt = tau == 1 ? th_cur : __ldg(ver(first_v + 1) + e);
            const float d0 = nxt - prev;
            st.vr = alpha * st.vr + one_m_a * g;
            st.va = alpha * st.va + one_m_a * g * g * d0;
        }
        float o = g;
        for (long long s = first_v; s < cur_v; ++s) {
            const float nxt = (s + 1 == cur_v) ? th_cur : __ldg(ver(s + 1) + e);
            o += lam * o * o * (nxt - prev);
            prev = nxt;
        }
        return o;
    }
}

// ---------------------------------------------------------------------------
// fused update: warp per parameter row, 4 consecutive columns per lane step
// (float4) when the row and every input row are 16-byte aligned.
// ---------------------------------------------------------------------------
template <int POLICY>
__global__ void __launch_bounds__(kThreads) update_kernel(const UpdArgs a) {
    __shared__ float sdel[kWarps][kMaxPending * kMaxBatch];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int gwarp = blockIdx.x * kWarps + wib;
    const int nwarps = gridDim.x * kWarps;
    const int K = a.K, B = a.B;
    const bool learn = a.eta > 0.f && a.v_r != nullptr;
    const RingVersions ver{a.ring, a.slot_floats, a.depth};
    const float* cur = ver(a.cur_version);
    float* dst = const_cast<float*>(ver(a.cur_version + 1));
    for (int row = gwarp; row < a.total_rows; row += nwarps) {
        int l = 0;
        while (l + 1 < a.n_layers && row >= a.L[l + 1].row0) ++l;
        const UpdLayer Ly = a.L[l];
        const int r = row - Ly.row0;
        __syncwarp();
        for (int i = lane; i < K * B; i += 32) {
            const int k = i / B, b = i % B;
            sdel[wib][i] = a.pend[k].stash[Ly.dlt_off + (size_t)b * Ly.out + r];
        }
        __syncwarp();
        const float* sd = sdel[wib];
        // input row of sample b for pending k
        auto xrow = [&](int k, int b) -> const float* {
            if (Ly.xin_off >= 0) return a.pend[k].stash + Ly.xin_off + (size_t)b * Ly.in;
            if (a.x0_gather) return a.pend[k].x0 + a.x0off[b];
            return a.pend[k].x0 + (size_t)b * a.x0_ld;
        };
        const size_t base = (size_t)Ly.woff + (size_t)r * Ly.in;
        bool vec = (Ly.in & 3) == 0 && (Ly.woff & 3) == 0;
        for (int k = 0; k < K && vec; ++k)
            for (int b = 0; b < B && vec; ++b) vec = aligned16(xrow(k, b));
        const int step = vec ? 4 : 1;
        for (int c0 = lane * step; c0 < Ly.in; c0 += 32 * step) {
            float gk[kMaxPending][4];
            for (int k = 0; k < K; ++k) {
                float g4[4] = {0.f, 0.f, 0.f, 0.f};
                for (int b = 0; b < B; ++b) {
                    const float* xr = xrow(k, b) + c0;
                    const float d = sd[k * B + b];
                    if (vec) {
                        const float4 x4 = __ldg(reinterpret_cast<const float4*>(xr));
                        g4[0] = fmaf(d, x4.x, g4[0]);
                        g4[1] = fmaf(d, x4.y, g4[1]);
                        g4[2] = fmaf(d, x4.z, g4[2]);
                        g4[3] = fmaf(d, x4.w, g4[3]);
                    } else {
                        g4[0] = fmaf(d, __ldg(xr), g4[0]);
                    }
                }
#pragma unroll
                for (int v = 0; v < 4; ++v) gk[k][v] = g4[v];
            }
            float th[4], ld[4] = {0.f, 0.f, 0.f, 0.f}, vr[4] = {0.f, 0.f, 0.f, 0.f}, va[4] = {0.f, 0.f, 0.f, 0.f},
                         gp[4] = {0.f, 0.f, 0.f, 0.f};
            const size_t e0 = base + c0;
            if (vec) {
                const float4 t4 = __ldg(reinterpret_cast<const float4*>(cur + e0));
                th[0] = t4.x; th[1] = t4.y; th[2] = t4.z; th[3] = t4.w;
                if (POLICY == 4) {
                    const float4 l4 = *reinterpret_cast<const float4*>(a.lam_d + e0);
                    ld[0] = l4.x; ld[1] = l4.y; ld[2] = l4.z; ld[3] = l4.w;
                    if (learn) {
                        const float4 r4 = *reinterpret_cast<const float4*>(a.v_r + e0);
                        const float4 a4 = *reinterpret_cast<const float4*>(a.v_a + e0);
                        vr[0] = r4.x; vr[1] = r4.y; vr[2] = r4.z; vr[3] = r4.w;
                        va[0] = a4.x; va[1] = a4.y; va[2] = a4.z; va[3] = a4.w;
                    }
                }
                if (POLICY == 2) {
                    const float4 p4 = *reinterpret_cast<const float4*>(a.gap + e0);
                    gp[0] = p4.x; gp[1] = p4.y; gp[2] = p4.z; gp[3] = p4.w;
                }
            } else {
                th[0] = __ldg(cur + e0);
                if (POLICY == 4) {
                    ld[0] = a.lam_d[e0];
                    if (learn) { vr[0] = a.v_r[e0]; va[0] = a.v_a[e0]; }
                }
                if (POLICY == 2) gp[0] = a.gap[e0];
            }
            float nt[4];
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                if (v >= step) break;
                ElemState st{ld[v], vr[v], va[v], gp[v]};
                float mean = 0.f;
                for (int k = 0; k < K; ++k)
                    mean += compensate_elem<POLICY>(gk[k][v], ver, a.pend[k].read_version, a.cur_version, e0 + v,
                                                    th[v], st, a.lambda0, a.alpha, a.eta, a.nu, learn);
                nt[v] = th[v] - a.step * mean;
                ld[v] = st.ld; vr[v] = st.vr; va[v] = st.va; gp[v] = st.gp;
            }
            if (vec) {
                *reinterpret_cast<float4*>(dst + e0) = make_float4(nt[0], nt[1], nt[2], nt[3]);
                if (POLICY == 4) {
                    *reinterpret_cast<float4*>(a.lam_d + e0) = make_float4(ld[0], ld[1], ld[2], ld[3]);
                    if (learn) {
                        *reinterpret_cast<float4*>(a.v_r + e0) = make_float4(vr[0], vr[1], vr[2], vr[3]);
                        *reinterpret_cast<float4*>(a.v_a + e0) = make_float4(va[0], va[1], va[2], va[3]);
                    }
                }
                if (POLICY == 2) *reinterpret_cast<float4*>(a.gap + e0) = make_float4(gp[0], gp[1], gp[2], gp[3]);
            } else {
                dst[e0] = nt[0];
                if (POLICY == 4) {
                    a.lam_d[e0] = ld[0];
                    if (learn) { a.v_r[e0] = vr[0]; a.v_a[e0] = va[0]; }
                }
                if (POLICY == 2) a.gap[e0] = gp[0];
            }
        }
        // bias element of this row (lane 0)
        if (lane == 0) {
            const size_t e = (size_t)Ly.boff + r;
            const float thc = __ldg(cur + e);
            ElemState st{0.f, 0.f, 0.f, 0.f};
            if (POLICY == 4) {
                st.ld = a.lam_d[e];
                if (learn) { st.vr = a.v_r[e]; st.va = a.v_a[e]; }
            }
            if (POLICY == 2) st.gp = a.gap[e];
            float mean = 0.f;
            for (int k = 0; k < K; ++k) {
                float g = 0.f;
                for (int b = 0; b < B; ++b) g += sd[k * B + b];
                mean += compensate_elem<POLICY>(g, ver, a.pend[k].read_version, a.cur_version, e, thc, st,
                                                a.lambda0, a.alpha, a.eta, a.nu, learn);
            }
            dst[e] = thc - a.step * mean;
            if (POLICY == 4) {
                a.lam_d[e] = st.ld;
                if (learn) { a.v_r[e] = st.vr; a.v_a[e] = st.va; }
            }
            if (POLICY == 2) a.gap[e] = st.gp;
        }
    }
}

// ---------------------------------------------------------------------------
// unit compensation kernel (flat, absolute lambda)
// ---------------------------------------------------------------------------
template <int POLICY>
__global__ void __launch_bounds__(kThreads) compensate_kernel(const CompArgs a) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    const bool learn = a.eta > 0.f && a.v_r != nullptr;
    const ListVersions ver{a.chain};
    const long long last = a.chain_len - 1;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < a.n; e += stride) {
        ElemState st{0.f, 0.f, 0.f, 0.f};
        if (POLICY == 4) {
            st.ld = a.lambda[e];
            if (learn) { st.vr = a.v_r[e]; st.va = a.v_a[e]; }
        }
        if (POLICY == 2) st.gp = a.gap[e];
        const float thc = a.chain[last][e];
        a.out[e] = compensate_elem<POLICY>(a.g[e], ver, 0, last, (size_t)e, thc, st,
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
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= a.F) return;
    double mu = a.mean[f], m2 = a.m2[f];
    unsigned long long cnt = a.count0;
    for (long long i = 0; i < a.n; ++i) {
        const double x = a.raw[i * a.F + f];
        ++cnt;
        const double d = __dsub_rn(x, mu);
        mu = __dadd_rn(mu, __ddiv_rn(d, (double)cnt));
        m2 = __dadd_rn(m2, __dmul_rn(d, __dsub_rn(x, mu)));
        const double var = cnt > 1 ? __ddiv_rn(m2, (double)(cnt - 1)) : 1.0;
        const double sd = __dsqrt_rn(var < 1e-8 ? 1e-8 : var);
        a.out[i * a.F + f] = (float)__ddiv_rn(__dsub_rn(x, mu), sd);
    }
    a.mean[f] = mu;
    a.m2[f] = m2;
}

} // namespace

void launch_fwd(const FwdArgs& a, cudaStream_t s) {
    bool vec = (a.in & 3) == 0 && aligned16(a.W);
    for (int b = 0; b < a.B && vec; ++b) vec = aligned16(a.X + a.xoff[b]);
    if (a.B <= 1) fwd_dispatch_vec<1, 1>(a, s, vec);
    else if (a.B <= 2) fwd_dispatch_vec<2, 2>(a, s, vec);
    else if (a.B <= 4) fwd_dispatch_vec<4, 2>(a, s, vec);
    else if (a.B <= 8) fwd_dispatch_vec<8, 2>(a, s, vec);
    else fwd_dispatch_vec<16, 2>(a, s, vec);
}

void launch_head(const HeadArgs& a, cudaStream_t s) {
    head_kernel<<<(a.B + kWarps - 1) / kWarps, kThreads, 0, s>>>(a);
}

int bwd_col_tiles(int in) { return (in + kBwdCols - 1) / kBwdCols; }

int bwd_row_splits(int in, int out) {
    const int tiles = bwd_col_tiles(in);
    int splits = (2 * 148 + tiles - 1) / tiles;
    const int max_by_rows = (out + 15) / 16;
    if (splits > max_by_rows) splits = max_by_rows;
    const int min_for_smem = (out + kBwdMaxRowsPerSplit - 1) / kBwdMaxRowsPerSplit;
    if (splits < min_for_smem) splits = min_for_smem;
    if (splits < 1) splits = 1;
    return splits;
}

void launch_bwd(const BwdArgs& a, cudaStream_t s) {
    dim3 grid(bwd_col_tiles(a.in), a.row_splits);
    if (a.B <= 1) bwd_kernel<1><<<grid, kBwdCols, 0, s>>>(a);
    else if (a.B <= 2) bwd_kernel<2><<<grid, kBwdCols, 0, s>>>(a);
    else if (a.B <= 4) bwd_kernel<4><<<grid, kBwdCols, 0, s>>>(a);
    else if (a.B <= 8) bwd_kernel<8><<<grid, kBwdCols, 0, s>>>(a);
    else bwd_kernel<16><<<grid, kBwdCols, 0, s>>>(a);
}

void launch_update(const UpdArgs& a, cudaStream_t s) {
    int grid = (a.total_rows + kWarps - 1) / kWarps;
    if (grid > 148 * 32) grid = 148 * 32;
    switch (a.policy) {
        case 0: update_kernel<0><<<grid, kThreads, 0, s>>>(a); break;
        case 1: update_kernel<1><<<grid, kThreads, 0, s>>>(a); break;
        case 2: update_kernel<2><<<grid, kThreads, 0, s>>>(a); break;
        case 3: update_kernel<3><<<grid, kThreads, 0, s>>>(a); break;
        default: update_kernel<4><<<grid, kThreads, 0, s>>>(a); break;
    }
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

void launch_normalize(const NormArgs& a, cudaStream_t s) {
    normalize_kernel<<<(a.F + 127) / 128, 128, 0, s>>>(a);
}

} // namespace fb200
