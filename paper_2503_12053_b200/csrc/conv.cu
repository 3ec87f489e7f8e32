// Convolutional layers of the ferret-b200 trainer (BASELINE config 3). The
// reference has no convolution; the CPU restatement these kernels are checked
// against is the test suite's conv restatement (dense reference arithmetic generalised:
// net.hpp:99-113 forward, learner.hpp:456-474 backward).
//
// Every op is an implicit GEMM — the im2col matrix is never materialised, the
// operand loaders gather straight from the NCHW activation rows in the stash:
//   fwd    C[c_out x B*HWo]   = W[c_out x c_in*k*k] . im2col(x)
//   dgrad  C[c_in  x B*HWi]   = W^T (per tap) . scatter(delta)        (transposed conv)
//   wgrad  C[c_out x c_in*k*k] = delta[c_out x B*HWo] . im2col(x)^T
// Two implementations: conv_mma_kernel (tcgen05 tensor cores, the default: 3xTF32
// in the fp32 parity mode, tf32 in the fast modes) and conv_gemm_kernel (SIMT
// FFMA, 64 x 64 CTA tiles, K in steps of 16 through shared memory, 4 x 4 fp32
// accumulators per thread; FERRET_CONV_TC=0). Grids with few tiles split K over
// blockIdx.z into a partial buffer, reduced in split order by a second kernel
// that also runs the epilogue, so results do not depend on scheduling (bitwise
// reproducible).
#include "kernels.cuh"
#include "umma.cuh"

#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

namespace fb200 {

namespace {

constexpr int TM = 64, TN = 64, TK = 16, NT = 256;
__device__ const float kConvOne = 1.0f;  // the B operand of the wgrad bias column (ConvArgs::bcol)

template <class Args>
void fill_spec(KernelSpec& k, const void* func, dim3 grid, dim3 block, const Args& a) {
    static_assert(sizeof(Args) <= sizeof(k.arg0), "kernel argument too large");
    k.func = func;
    k.grid = grid;
    k.block = block;
    k.smem = 0;
    std::memcpy(k.arg0, &a, sizeof(Args));
    k.nargs = 1;
}

// the B-operand column a thread loads, decomposed once
struct Col {
    int ok;
    int b, y, x;               // fwd: (b, oh, ow); dgrad: (b, ih, iw)
    int ci, kh, kw;            // wgrad: (ci, kh, kw)
    const float* row;          // fwd / dgrad: the sample's row (x or delta)
};

template <int MODE>
__device__ __forceinline__ Col make_col(const ConvArgs& a, int n) {
    Col c{};
    c.ok = n < a.N;
    if (!c.ok) return c;
    if (MODE == kConvFwd) {
        const int hw = a.ho * a.wo;
        c.b = n / hw;
        const int pix = n - c.b * hw;
        c.y = pix / a.wo;
        c.x = pix - c.y * a.wo;
        const size_t in_w = (size_t)a.ci * a.hi * a.wi;
        c.row = a.X + (a.xidx ? (size_t)__ldg(a.xidx + c.b) : (size_t)c.b) * in_w;
    } else if (MODE == kConvDgrad) {
        const int hw = a.hi * a.wi;
        c.b = n / hw;
        const int pix = n - c.b * hw;
        c.y = pix / a.wi;
        c.x = pix - c.y * a.wi;
        c.row = a.D + (size_t)c.b * a.co * a.ho * a.wo;
    } else {
        const int kk = a.k * a.k;
        c.ci = n / kk;
        const int r = n - c.ci * kk;
        c.kh = r / a.k;
        c.kw = r - c.kh * a.k;
    }
    return c;
}

template <int MODE>
__device__ __forceinline__ float load_a(const ConvArgs& a, int m, int k) {
    if (MODE == kConvFwd) return __ldg(a.W + (size_t)m * a.K + k);
    if (MODE == kConvDgrad) {
        const int kk = a.k * a.k;
        const int co = k / kk, r = k - co * kk;
        return __ldg(a.W + ((size_t)co * a.ci + m) * kk + r);
    }
    const int hw = a.ho * a.wo;
    const int b = k / hw, pix = k - b * hw;
    return __ldg(a.D + ((size_t)b * a.co + m) * hw + pix);
}

template <int MODE>
__device__ __forceinline__ float load_b(const ConvArgs& a, const Col& c, int k) {
    if (MODE == kConvFwd) {
        const int kk = a.k * a.k;
        const int ci = k / kk, r = k - ci * kk;
        const int kh = r / a.k, kw = r - kh * a.k;
        const int ih = c.y * a.s - a.p + kh, iw = c.x * a.s - a.p + kw;
        if ((unsigned)ih >= (unsigned)a.hi || (unsigned)iw >= (unsigned)a.wi) return 0.f;
        return __ldg(c.row + ((size_t)ci * a.hi + ih) * a.wi + iw);
    }
    if (MODE == kConvDgrad) {
        const int kk = a.k * a.k;
        const int co = k / kk, r = k - co * kk;
        const int kh = r / a.k, kw = r - kh * a.k;
        const int th = c.y + a.p - kh, tw = c.x + a.p - kw;
        if (th < 0 || tw < 0) return 0.f;
        const int oh = th / a.s, ow = tw / a.s;
        if (oh * a.s != th || ow * a.s != tw || oh >= a.ho || ow >= a.wo) return 0.f;
        return __ldg(c.row + ((size_t)co * a.ho + oh) * a.wo + ow);
    }
    const int hw = a.ho * a.wo;
    const int b = k / hw, pix = k - b * hw;
    const int oh = pix / a.wo, ow = pix - oh * a.wo;
    const int ih = oh * a.s - a.p + c.kh, iw = ow * a.s - a.p + c.kw;
    if ((unsigned)ih >= (unsigned)a.hi || (unsigned)iw >= (unsigned)a.wi) return 0.f;
    const size_t in_w = (size_t)a.ci * a.hi * a.wi;
    const float* row = a.X + (a.xidx ? (size_t)__ldg(a.xidx + b) : (size_t)b) * in_w;
    return __ldg(row + ((size_t)c.ci * a.hi + ih) * a.wi + iw);
}

// bias + shortcut + activation (fwd), skip + ReLU mask (dgrad), plain store (wgrad)
template <int MODE>
__device__ __forceinline__ void epilogue(const ConvArgs& a, int m, int n, float v) {
    if (MODE == kConvWgrad) {
        if (a.bcol) a.Y[n == a.N - 1 ? (size_t)a.M * (a.N - 1) + m : (size_t)m * (a.N - 1) + n] = v;
        else a.Y[(size_t)m * a.N + n] = v;
        return;
    }
    if (MODE == kConvFwd) {
        const int hw = a.ho * a.wo;
        const int b = n / hw, pix = n - b * hw;
        v += __ldg(a.bias + m);
        if (a.res && m < a.rc) {  // option-A shortcut: subsample by the stride, channels [0, rc)
            const int oh = pix / a.wo, ow = pix - oh * a.wo, st = a.rh / a.ho;
            v += __ldg(a.res + ((size_t)b * a.rc + m) * a.rh * a.rw + (size_t)(oh * st) * a.rw + ow * st);
        }
        if (a.relu) v = v > 0.f ? v : 0.f;
        a.Y[((size_t)b * a.co + m) * hw + pix] = v;
        return;
    }
    const int hw = a.hi * a.wi;
    const int b = n / hw, pix = n - b * hw;
    if (a.res) {  // S^T(delta of the residual layer above): its strided positions
        const int ih = pix / a.wi, iw = pix - ih * a.wi, st = a.hi / a.rh;
        if (ih % st == 0 && iw % st == 0)
            v += __ldg(a.res + ((size_t)b * a.rc + m) * a.rh * a.rw + (size_t)(ih / st) * a.rw + iw / st);
    }
    const size_t o = ((size_t)b * a.ci + m) * hw + pix;
    if (a.mask && !(__ldg(a.mask + o) > 0.f)) v = 0.f;
    a.Y[o] = v;
}

template <int MODE>
__global__ void __launch_bounds__(NT) conv_gemm_kernel(const ConvArgs a) {
    FB_PDL_ENTRY();
    __shared__ __align__(16) float As[TK][TM];
    __shared__ __align__(16) float Bs[TK][TN];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
    const int kbeg = blockIdx.z * a.kchunk;
    const int kend = min(a.K, kbeg + a.kchunk);
    // loaders: A row am (4 consecutive k from ka), B column bn (k rows kb + 4 i)
    const int am = tid >> 2, ka = (tid & 3) * 4;
    const int bn = tid & 63, kb = tid >> 6;
    const bool arow = m0 + am < a.M;
    const Col col = make_col<MODE>(a, n0 + bn);
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
    float ra[4], rb[4];
    auto fetch = [&](int k0) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int k = k0 + ka + i;
            ra[i] = (arow && k < kend) ? load_a<MODE>(a, m0 + am, k) : 0.f;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int k = k0 + kb + 4 * i;
            rb[i] = (col.ok && k < kend) ? load_b<MODE>(a, col, k) : 0.f;
        }
    };
    fetch(kbeg);
    for (int k0 = kbeg; k0 < kend; k0 += TK) {
        __syncthreads();
#pragma unroll
        for (int i = 0; i < 4; ++i) As[ka + i][am] = ra[i];
#pragma unroll
        for (int i = 0; i < 4; ++i) Bs[kb + 4 * i][bn] = rb[i];
        __syncthreads();
        if (k0 + TK < kend) fetch(k0 + TK);  // next tile's loads in flight during the FMAs
#pragma unroll
        for (int kk = 0; kk < TK; ++kk) {
            const float4 av = *reinterpret_cast<const float4*>(&As[kk][ty * 4]);
            const float4 bv = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
            const float am4[4] = {av.x, av.y, av.z, av.w};
            const float bn4[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(am4[i], bn4[j], acc[i][j]);
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int m = m0 + ty * 4 + i;
        if (m >= a.M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int n = n0 + tx * 4 + j;
            if (n >= a.N) continue;
            if (a.splits > 1)
                a.partial[((size_t)blockIdx.z * a.M + m) * a.N + n] = acc[i][j];
            else
                epilogue<MODE>(a, m, n, acc[i][j]);
        }
    }
}

// ordered sum of the K-split partials, then the epilogue. Few splits: a thread
// per output, splits in order. Many splits (weight gradients of small layers:
// up to ~150 partials over few outputs): a warp per output, lane l summing splits
// l, l+32, ... in order, then a fixed butterfly — deterministic either way.
constexpr int kWarpReduceSplits = 16;
constexpr long long kWarpReduceMaxOutputs = 32768;  // larger outputs: coalesced thread-per-output wins
__host__ __device__ inline bool warp_reduce(const ConvArgs& a) {
    return a.splits >= kWarpReduceSplits && (long long)a.M * a.N <= kWarpReduceMaxOutputs;
}
template <int MODE>
__global__ void __launch_bounds__(NT) conv_reduce_kernel(const ConvArgs a) {
    FB_PDL_ENTRY();
    const size_t mn = (size_t)a.M * a.N;
    if (warp_reduce(a)) {
        const int lane = threadIdx.x & 31;
        for (size_t i = ((size_t)blockIdx.x * NT + threadIdx.x) >> 5; i < mn; i += ((size_t)gridDim.x * NT) >> 5) {
            float v = 0.f;
            for (int s = lane; s < a.splits; s += 32) v += __ldg(a.partial + (size_t)s * mn + i);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0) {
                const int m = (int)(i / a.N), n = (int)(i - (size_t)m * a.N);
                epilogue<MODE>(a, m, n, v);
            }
        }
        return;
    }
    for (size_t i = (size_t)blockIdx.x * NT + threadIdx.x; i < mn; i += (size_t)gridDim.x * NT) {
        float v = 0.f;
        for (int s = 0; s < a.splits; ++s) v += __ldg(a.partial + (size_t)s * mn + i);
        const int m = (int)(i / a.N), n = (int)(i - (size_t)m * a.N);
        epilogue<MODE>(a, m, n, v);
    }
}

// gb[co] = sum_b sum_pix D[b][co][pix]: one CTA per channel, thread t summing pixels
// t, t + 256, ... of every sample in order, then a fixed butterfly + ordered warp sums
// (deterministic). (gb = a.Y)
__global__ void __launch_bounds__(NT) conv_bgrad_kernel(const ConvArgs a) {
    FB_PDL_ENTRY();
    __shared__ float part[NT / 32];
    const int ch = blockIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int hw = a.ho * a.wo;
    // four independent accumulators (samples b mod 4) so the loads pipeline; combined in order
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int b0 = 0; b0 < a.B; b0 += 4) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (b0 + q >= a.B) break;
            const float* d = a.D + ((size_t)(b0 + q) * a.co + ch) * hw;
            for (int p = threadIdx.x; p < hw; p += NT) acc[q] += __ldg(d + p);
        }
    }
    float v = (acc[0] + acc[1]) + (acc[2] + acc[3]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) part[w] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        float sum = 0.f;
#pragma unroll
        for (int k = 0; k < NT / 32; ++k) sum += part[k];
        a.Y[ch] = sum;
    }
}

__global__ void __launch_bounds__(NT) gap_kernel(const PoolMeanArgs a) {
    FB_PDL_ENTRY();
    const int i = blockIdx.x * NT + threadIdx.x;
    if (i >= a.B * a.C) return;
    const int b = i / a.C, c = i - b * a.C;
    const float* x = a.X + (a.xidx ? (size_t)__ldg(a.xidx + b) : (size_t)b) * a.C * a.HW + (size_t)c * a.HW;
    float s = 0.f;
    for (int p = 0; p < a.HW; ++p) s += __ldg(x + p);
    a.Y[i] = s / (float)a.HW;
}

__global__ void __launch_bounds__(NT) ungap_kernel(const PoolMeanArgs a) {
    FB_PDL_ENTRY();
    const size_t n = (size_t)a.B * a.C * a.HW;
    for (size_t i = (size_t)blockIdx.x * NT + threadIdx.x; i < n; i += (size_t)gridDim.x * NT) {
        float v = __ldg(a.dY + i / a.HW) / (float)a.HW;
        if (a.mask && !(__ldg(a.mask + i) > 0.f)) v = 0.f;
        a.dX[i] = v;
    }
}

// ---------------------------------------------------------------------------
// Tensor-core implicit GEMM (tcgen05): 128 x 128 output tile per CTA, fp32
// accumulator in 128 TMEM columns. 8 producer warps gather the A and B operands
// of each 128-byte K atom straight from the activations / weights with cp.async
// (4-byte element copies with zero fill for padding; 16-byte copies for the
// contiguous rows of the tap-major prepared weights and of weight-gradient deltas)
// into a 3-5 stage smem ring, K-major with the 128-byte swizzle; one thread issues
// the MMAs (M 128, N 128, 4 per atom) and frees each stage with tcgen05.commit.
// 3xTF32 (the fp32 parity mode) adds a tf32 lo tile per operand (lo = x - hi,
// written by the thread that copied x; hi is the raw operand, which kind::tf32
// truncates; stage layout A, B, B lo, A lo) and issues hi_A x [hi_B; lo_B] as one
// N = 256 MMA into 256 TMEM columns (halves summed in the epilogue) plus lo_A x hi_B. The epilogue reads TMEM
// (tcgen05.ld), stages the tile through smem so global stores are coalesced along
// pixels, then runs the SIMT kernel's epilogue (bias / shortcut / ReLU, skip /
// mask) or writes the split-K partial (reduced in split order by conv_reduce_kernel).
// ---------------------------------------------------------------------------
// warp 0: TMEM + MMA issue; warps 1-8: producers (cp.async gathers), epilogue
// Producer lag: a thread publishes atom i - LAG after issuing the copies of atom i. With
// LAG = NST - 1 the MMA only ever had one published atom (issue of atom i waits on the MMA of
// atom i - NST, publication of i - NST + 1 follows it): lag NST / 2 lets published atoms
// queue for the MMA (C3 3.3-3.5k -> 3.65k samples/s; lag 1 measured the same)
#ifndef FERRET_CONV_LAG_DIV
#define FERRET_CONV_LAG_DIV 2
#endif
#define FERRET_CONV_LAG (NST / FERRET_CONV_LAG_DIV > 0 ? NST / FERRET_CONV_LAG_DIV : 1)
constexpr int kCP = 256;
constexpr int kCT = 32 + kCP;
// smem ring depth: 3 x 64 KB (3xTF32: raw + lo operands) or 3 x 32 KB (tf32)
// (3 x 32 KB for tf32 keeps two CTAs per SM resident — 2 x 97 KB smem, 2 x 288 x <= 107
// registers — so one CTA's producer / MMA handshake overlaps the other's: +4 % over 5 stages
// at one CTA per SM)
__host__ __device__ constexpr int conv_stages(bool split) { return 3; }
constexpr int kCTile = 16384;  // 128 rows x 128 bytes

// Operand element sources of the tensor-core kernel (nullptr = zero: padding,
// out of range). Tap-major (ConvArgs::kt): k = tap * C + c, C = the channel count of
// the operand that is summed over (fwd: c_in; dgrad: c_out), C % atom == 0.
template <int MODE, int NE>
__device__ __forceinline__ void locate_a_tm(const ConvArgs& a, int m, bool ok, int k0, const float* (&P)[NE]) {
    const int kk = a.k * a.k;
    const int C = MODE == kConvFwd ? a.ci : a.co;
    const int tap = k0 / C, c0 = k0 - tap * C;
    if (!ok) {
#pragma unroll
        for (int e = 0; e < NE; ++e) P[e] = nullptr;
        return;
    }
    // fwd: W[m][c][tap]; dgrad: W[c][m][tap]
    const float* w = MODE == kConvFwd ? a.W + ((size_t)m * a.ci + c0) * kk + tap : a.W + ((size_t)c0 * a.ci + m) * kk + tap;
    const size_t step = MODE == kConvFwd ? (size_t)kk : (size_t)a.ci * kk;
#pragma unroll
    for (int e = 0; e < NE; ++e) P[e] = w + e * step;
}

template <int MODE, int NE>
__device__ __forceinline__ void locate_b_tm(const ConvArgs& a, const Col& c, int k0, const float* (&P)[NE]) {
    const int C = MODE == kConvFwd ? a.ci : a.co;
    const int tap = k0 / C, c0 = k0 - tap * C;
    const int kh = tap / a.k, kw = tap - kh * a.k;
    const float* src = nullptr;
    size_t step = 0;
    if (c.ok) {
        if (MODE == kConvFwd) {
            const int ih = c.y * a.s - a.p + kh, iw = c.x * a.s - a.p + kw;
            if ((unsigned)ih < (unsigned)a.hi && (unsigned)iw < (unsigned)a.wi) {
                src = c.row + ((size_t)c0 * a.hi + ih) * a.wi + iw;
                step = (size_t)a.hi * a.wi;
            }
        } else {
            int th = c.y + a.p - kh, tw = c.x + a.p - kw;
            bool in = th >= 0 && tw >= 0;
            if (a.s == 2) {
                in = in && !((th | tw) & 1);
                th >>= 1;
                tw >>= 1;
            } else if (a.s != 1) {
                in = in && th % a.s == 0 && tw % a.s == 0;
                th /= a.s;
                tw /= a.s;
            }
            if (in && th < a.ho && tw < a.wo) {
                src = c.row + ((size_t)c0 * a.ho + th) * a.wo + tw;
                step = (size_t)a.ho * a.wo;
            }
        }
    }
    if (!src) {
#pragma unroll
        for (int e = 0; e < NE; ++e) P[e] = nullptr;
        return;
    }
#pragma unroll
    for (int e = 0; e < NE; ++e) P[e] = src + e * step;
}

template <int MODE, int NE>
__device__ __forceinline__ void locate_a(const ConvArgs& a, int m, bool ok, int k0, const float* (&P)[NE]) {
    if (!ok) {
#pragma unroll
        for (int e = 0; e < NE; ++e) P[e] = nullptr;
        return;
    }
    if (MODE == kConvFwd) {  // W row m, contiguous in k
        const float* w = a.W + (size_t)m * a.K;
#pragma unroll
        for (int e = 0; e < NE; ++e) P[e] = k0 + e < a.K ? w + k0 + e : nullptr;
    } else if (MODE == kConvDgrad) {  // W[co][m][tap], k = co * kk + tap
        const int kk = a.k * a.k;
        const int co = k0 / kk;
        int r = k0 - co * kk;
        const float* w = a.W + ((size_t)co * a.ci + m) * kk;
        const size_t jump = (size_t)a.ci * kk;
#pragma unroll
        for (int e = 0; e < NE; ++e) {
            P[e] = k0 + e < a.K ? w + r : nullptr;
            if (++r == kk) {
                r = 0;
                w += jump;
            }
        }
    } else {  // delta[b][m][pix], k = b * HWo + pix
        const int hw = a.ho * a.wo;
        const int b = k0 / hw;
        int pix = k0 - b * hw;
        const float* d = a.D + ((size_t)b * a.co + m) * hw;
        const size_t jump = (size_t)a.co * hw;
#pragma unroll
        for (int e = 0; e < NE; ++e) {
            P[e] = k0 + e < a.K ? d + pix : nullptr;
            if (++pix == hw) {
                pix = 0;
                d += jump;
            }
        }
    }
}

template <int MODE, int NE>
__device__ __forceinline__ void locate_b(const ConvArgs& a, const Col& c, int k0, const float* (&P)[NE]) {
    if (!c.ok) {
#pragma unroll
        for (int e = 0; e < NE; ++e) P[e] = nullptr;
        return;
    }
    if (MODE == kConvFwd || MODE == kConvDgrad) {
        // k = ch * kk + kh * k + kw (fwd: ch = c_in of x; dgrad: ch = c_out of delta)
        const int kk = a.k * a.k;
        int ch = k0 / kk;
        const int r = k0 - ch * kk;
        int kh = r / a.k, kw = r - kh * a.k;
#pragma unroll
        for (int e = 0; e < NE; ++e) {
            const float* x = nullptr;
            if (k0 + e < a.K) {
                if (MODE == kConvFwd) {
                    const int ih = c.y * a.s - a.p + kh, iw = c.x * a.s - a.p + kw;
                    if ((unsigned)ih < (unsigned)a.hi && (unsigned)iw < (unsigned)a.wi)
                        x = c.row + ((size_t)ch * a.hi + ih) * a.wi + iw;
                } else {
                    int th = c.y + a.p - kh, tw = c.x + a.p - kw;
                    bool in = th >= 0 && tw >= 0;
                    if (a.s == 2) {
                        in = in && !((th | tw) & 1);
                        th >>= 1;
                        tw >>= 1;
                    } else if (a.s != 1) {
                        in = in && th % a.s == 0 && tw % a.s == 0;
                        th /= a.s;
                        tw /= a.s;
                    }
                    if (in && th < a.ho && tw < a.wo) x = c.row + ((size_t)ch * a.ho + th) * a.wo + tw;
                }
            }
            P[e] = x;
            if (++kw == a.k) {
                kw = 0;
                if (++kh == a.k) {
                    kh = 0;
                    ++ch;
                }
            }
        }
    } else {  // wgrad: column (ci, kh, kw) fixed; k = b * HWo + oh * wo + ow
        if (a.bcol && c.ci >= a.ci) {  // the bias column: B = 1 for every k (the bias gradient)
#pragma unroll
            for (int e = 0; e < NE; ++e) P[e] = k0 + e < a.K ? &kConvOne : nullptr;
            return;
        }
        const int hw = a.ho * a.wo;
        int b = k0 / hw;
        const int pix = k0 - b * hw;
        int oh = pix / a.wo, ow = pix - oh * a.wo;
        const size_t in_w = (size_t)a.ci * a.hi * a.wi;
        const size_t coff = (size_t)c.ci * a.hi * a.wi;
        auto rowp = [&](int bb) {
            return a.X + (a.xidx ? (size_t)__ldg(a.xidx + bb) : (size_t)bb) * in_w + coff;
        };
        const float* row = b < a.B ? rowp(b) : a.X;
#pragma unroll
        for (int e = 0; e < NE; ++e) {
            const float* x = nullptr;
            if (k0 + e < a.K) {
                const int ih = oh * a.s - a.p + c.kh, iw = ow * a.s - a.p + c.kw;
                if ((unsigned)ih < (unsigned)a.hi && (unsigned)iw < (unsigned)a.wi) x = row + (size_t)ih * a.wi + iw;
            }
            P[e] = x;
            if (++ow == a.wo) {
                ow = 0;
                if (++oh == a.ho) {
                    oh = 0;
                    if (++b < a.B) row = rowp(b);
                }
            }
        }
    }
}

template <int MODE, int ES, bool SPLIT>
__global__ void __launch_bounds__(kCT, SPLIT ? 1 : 2) conv_mma_kernel(const __grid_constant__ ConvArgs a) {
    FB_PDL_ENTRY();
    constexpr int KA = 128 / ES;  // K elements per atom
    constexpr int UK = 32 / ES;   // K per MMA
    constexpr int CE = 16 / ES;   // elements per 16-byte chunk
    constexpr bool TF32 = ES == 4;
    constexpr int STAGE = kCTile * 2 * (SPLIT ? 2 : 1);  // A, B (then A lo, B lo)
    constexpr int NST = conv_stages(SPLIT);
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(base + NST * STAGE);
    uint64_t* empty = full + NST;
    uint64_t* done = empty + NST;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m0 = blockIdx.y * 128, n0 = blockIdx.x * 128;
    const int katoms = (a.K + KA - 1) / KA;
    const int a_lo = blockIdx.z * a.apc;
    const int na = max(0, min(katoms, a_lo + a.apc) - a_lo);
    // phase stamps: 0 start, 1 setup done, 2 first atom published, 3 first MMA issued,
    // 4 last MMA committed, 5 accumulator ready (epilogue), 6 stores done
    unsigned long long* stamp =
        a.stamps ? a.stamps + (((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) * 8 : nullptr;
    auto tick = [&](int k) {
        if (stamp) {
            unsigned long long tt;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
            stamp[k] = tt;
        }
    };
    if (threadIdx.x == 0) tick(0);

    if (threadIdx.x == 0) {
        for (int s = 0; s < NST; ++s) {
            mbar_init(full + s, kCP);
            mbar_init(empty + s, 1);
        }
        mbar_init(done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(SPLIT ? 256 : 128));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;
    if (threadIdx.x == 0) tick(1);

    if (warp == 0) {
        if (lane == 0 && na > 0) {
            // instruction descriptor: D f32, A/B tf32 (2) or bf16 (1), both K-major, N >> 3, M >> 4
            const uint32_t fmt = TF32 ? 2u : 1u;
            const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
            for (int i = 0; i < na; ++i) {
                const int s = i % NST;
                mbar_wait(full + s, (i / NST) & 1);
                if (i == 0) tick(3);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t abase = smem_u32(base + s * STAGE);
                const uint32_t bbase = abase + kCTile;
#pragma unroll
                for (int k = 0; k < KA / UK; ++k) {
                    const uint64_t ad = smem_desc(abase + k * 32, 16, 1024);
                    const uint64_t bd = smem_desc(bbase + k * 32, 16, 1024);
                    if constexpr (SPLIT) {
                        // hi_A x [hi_B; lo_B]: B hi and B lo are one N = 256 operand (stage layout A, B,
                        // B lo, A lo), accumulator columns 0-127 and 128-255 summed in the epilogue;
                        // then + lo_A hi_B (N = 128): 8 MMAs per atom instead of 12
                        const uint32_t idesc256 = (idesc & ~(0x3Fu << 17)) | ((256u >> 3) << 17);
                        umma(tmem, ad, bd, idesc256, (i > 0 || k > 0) ? 1u : 0u, TF32);
                        umma(tmem, smem_desc(abase + 3 * kCTile + k * 32, 16, 1024), bd, idesc, 1u, TF32);
                    } else {
                        umma(tmem, ad, bd, idesc, (i > 0 || k > 0) ? 1u : 0u, TF32);
                    }
                }
                umma_commit(empty + s);
            }
            umma_commit(done);
            tick(4);
        }
    } else {
        // ---- producers: thread t owns operand row r (A: output row m0 + r; B: GEMM
        // column n0 + r) and 16-byte chunks jh .. jh + 3 of every atom. Each element
        // is one 4-byte cp.async (zero-filled where the operand is padding), so a
        // thread keeps D = NST - 1 atoms of copies in flight instead of waiting on
        // its loads; an atom is published (3xTF32: after the thread splits its own
        // elements into tf32 hi / lo) once the thread's copies of it have landed.
        constexpr int D = FERRET_CONV_LAG;
        const int t = threadIdx.x - 32, r = t >> 1, jh = (t & 1) * 4;
        const bool arow = m0 + r < a.M;
        const Col col = make_col<MODE>(a, n0 + r);
        const int sw = r & 7;
        const int rbase = (r >> 3) * 1024 + (r & 7) * 128;
        auto issue = [&](unsigned char* X, const float* const (&P)[4 * CE]) {
#pragma unroll
            for (int e = 0; e < 4 * CE; ++e) {
                const uint32_t dst = smem_u32(X + rbase + (((jh + e / CE) ^ sw) << 4) + (e % CE) * 4);
                const float* src = P[e] ? P[e] : a.W;
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(P[e] ? 4 : 0)
                             : "memory");
            }
        };
        // contiguous A rows (see below) are copied with 8 lanes per row: rows q * 32 + t / 8,
        // chunk t % 8; everything else with the thread's own row r, chunks jh .. jh + 3
        const bool arun = MODE == kConvWgrad ? (a.ho * a.wo) % CE == 0 : (a.kt && a.Wt != nullptr);
        const int ja = t & 7;
        // lo = x - hi goes 2 tiles further; hi stays implicit: kind::tf32 reads the raw fp32
        // operand and drops its low 13 mantissa bits, i.e. multiplies exactly tf32_hi(x)
        // (checked by the 3xTF32 unit tests at 2e-6; writing hi back cost 2.7 % of C3)
        auto split16 = [&](unsigned char* p, int lo_off) {
            const float4 x = *reinterpret_cast<const float4*>(p);
            const float4 hi = make_float4(tf32_hi(x.x), tf32_hi(x.y), tf32_hi(x.z), tf32_hi(x.w));
            *reinterpret_cast<float4*>(p + lo_off) = make_float4(x.x - hi.x, x.y - hi.y, x.z - hi.z, x.w - hi.w);
        };
        // once the thread's own copies of atom i have landed: (3xTF32) split exactly the
        // elements this thread copied, then publish its share of the atom
        auto publish = [&](int i) {
            const int s = i % NST;
            if constexpr (SPLIT) {
                unsigned char* A = base + s * STAGE;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    if (arun) {
                        const int ra = q * 32 + (t >> 3);
                        split16(A + (ra >> 3) * 1024 + (ra & 7) * 128 + ((ja ^ (ra & 7)) << 4), 3 * kCTile);
                    } else {
                        split16(A + rbase + (((jh + q) ^ sw) << 4), 3 * kCTile);
                    }
                    split16(A + kCTile + rbase + (((jh + q) ^ sw) << 4), kCTile);
                }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(full + s)) : "memory");
            if (i == 0 && t == 0) tick(2);
        };
        // A rows that are contiguous runs: the prepared tap-major weights (fwd / dgrad) or the
        // delta rows of a weight gradient (HWo % 4 == 0) go as 16-byte copies with 8 lanes per
        // 128-byte row, so a warp instruction touches 4 lines (one row per lane would touch 32)
        for (int i = 0; i < na; ++i) {
            const int s = i % NST;
            if (i >= NST) mbar_wait(empty + s, ((i / NST) - 1) & 1);
            unsigned char* sa = base + s * STAGE;
            const int k0 = (a_lo + i) * KA + jh * CE;  // the thread's 4 chunks are 4 * CE consecutive k
            const float* P[4 * CE];
            if (arun) {
                const int ka = (a_lo + i) * KA + ja * CE;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int ra = q * 32 + (t >> 3), m = m0 + ra;
                    const float* src = nullptr;
                    if (m < a.M && ka < a.K) {
                        if (MODE == kConvWgrad) {
                            const int hw = a.ho * a.wo, b = ka / hw;
                            src = a.D + ((size_t)b * a.co + m) * hw + (ka - b * hw);
                        } else {
                            src = a.Wt + (size_t)m * a.K + ka;
                        }
                    }
                    const uint32_t dst = smem_u32(sa + (ra >> 3) * 1024 + (ra & 7) * 128 + ((ja ^ (ra & 7)) << 4));
                    if (!(a.dbg & 1))
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src ? src : a.W),
                                     "r"(src ? 16 : 0)
                                     : "memory");
                }
            } else {
                if (MODE != kConvWgrad && a.kt)
                    locate_a_tm<MODE, 4 * CE>(a, m0 + r, arow, k0, P);
                else
                    locate_a<MODE, 4 * CE>(a, m0 + r, arow, k0, P);
                issue(sa, P);
            }
            if (!(a.dbg & 2)) {
                if (MODE != kConvWgrad && a.kt)
                    locate_b_tm<MODE, 4 * CE>(a, col, k0, P);
                else
                    locate_b<MODE, 4 * CE>(a, col, k0, P);
                issue(sa + kCTile, P);
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
            if (i >= D) {
                asm volatile("cp.async.wait_group %0;" ::"n"(D) : "memory");
                publish(i - D);
            }
        }
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        for (int i = max(0, na - D); i < na; ++i) publish(i);
        // ---- epilogue: warps 1-4 move the accumulator (TMEM lane quadrant warp % 4)
        // into a padded smem tile; then all producers store it along pixels
        float* T = reinterpret_cast<float*>(base);  // 128 x 129 floats, over the drained ring
        if (warp <= 4) {
            const int q = warp & 3, row = q * 32 + lane;
            if (na > 0) {
                mbar_wait(done, 0);
                if (warp == 1 && lane == 0) tick(5);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    float v[16];
                    tmem_ld16(tmem + (static_cast<uint32_t>(q * 32) << 16) + c * 16, v);
                    if constexpr (SPLIT) {  // + hi_A lo_B (accumulator columns 128-255)
                        float w[16];
                        tmem_ld16(tmem + (static_cast<uint32_t>(q * 32) << 16) + 128 + c * 16, w);
#pragma unroll
                        for (int e = 0; e < 16; ++e) v[e] += w[e];
                    }
#pragma unroll
                    for (int e = 0; e < 16; ++e) T[row * 129 + c * 16 + e] = v[e];
                }
            } else {
                for (int c = 0; c < 128; ++c) T[row * 129 + c] = 0.f;
            }
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kCP) : "memory");
        // the thread's column n is fixed (stride 256 = two rows of 128): its sample /
        // pixel decomposition is done once, each row m is then one strided step
        const int nn = t & 127, n = n0 + nn;
        if (n < a.N) {
            const int mstart = t >> 7;
            if (a.splits > 1) {
                float* dst = a.partial + (size_t)blockIdx.z * a.M * a.N + n;
                for (int mm = mstart; mm < 128 && m0 + mm < a.M; mm += 2)
                    dst[(size_t)(m0 + mm) * a.N] = T[mm * 129 + nn];
            } else if (MODE == kConvWgrad) {
                // with the bias column (bcol) the weights are M x (N - 1) and the bias follows them
                const size_t ldw = a.bcol ? (size_t)(a.N - 1) : (size_t)a.N;
                const bool bias_col = a.bcol && n == a.N - 1;
                for (int mm = mstart; mm < 128 && m0 + mm < a.M; mm += 2)
                    a.Y[bias_col ? (size_t)a.M * ldw + m0 + mm : (size_t)(m0 + mm) * ldw + n] = T[mm * 129 + nn];
            } else if (MODE == kConvFwd) {
                const int hw = a.ho * a.wo, b = n / hw, pix = n - b * hw;
                float* y = a.Y + (size_t)b * a.co * hw + pix;
                const float* rs = nullptr;
                size_t rstep = 0;
                if (a.res) {
                    const int oh = pix / a.wo, ow = pix - oh * a.wo, st = a.rh / a.ho;
                    rstep = (size_t)a.rh * a.rw;
                    rs = a.res + (size_t)b * a.rc * rstep + (size_t)(oh * st) * a.rw + ow * st;
                }
                for (int mm = mstart; mm < 128 && m0 + mm < a.M; mm += 2) {
                    const int m = m0 + mm;
                    float v = T[mm * 129 + nn] + __ldg(a.bias + m);
                    if (rs && m < a.rc) v += __ldg(rs + (size_t)m * rstep);
                    if (a.relu) v = v > 0.f ? v : 0.f;
                    y[(size_t)m * hw] = v;
                }
            } else {  // dgrad
                const int hw = a.hi * a.wi, b = n / hw, pix = n - b * hw;
                const size_t o0 = (size_t)b * a.ci * hw + pix;
                const float* rs = nullptr;
                size_t rstep = 0;
                if (a.res) {
                    const int ih = pix / a.wi, iw = pix - ih * a.wi, st = a.hi / a.rh;
                    if (ih % st == 0 && iw % st == 0) {
                        rstep = (size_t)a.rh * a.rw;
                        rs = a.res + (size_t)b * a.rc * rstep + (size_t)(ih / st) * a.rw + iw / st;
                    }
                }
                for (int mm = mstart; mm < 128 && m0 + mm < a.M; mm += 2) {
                    const int m = m0 + mm;
                    const size_t o = o0 + (size_t)m * hw;
                    float v = T[mm * 129 + nn];
                    if (rs) v += __ldg(rs + (size_t)m * rstep);
                    if (a.mask && !(__ldg(a.mask + o) > 0.f)) v = 0.f;
                    a.Y[o] = v;
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) tick(6);
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(SPLIT ? 256 : 128));
    }
}

template <int MODE, int ES, bool SPLIT>
const void* conv_mma_func(size_t& smem) {
    smem = (size_t)conv_stages(SPLIT) * kCTile * 2 * (SPLIT ? 2 : 1) + 1024 + 128;
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(reinterpret_cast<const void*>(&conv_mma_kernel<MODE, ES, SPLIT>),
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured = true;
    }
    return reinterpret_cast<const void*>(&conv_mma_kernel<MODE, ES, SPLIT>);
}

template <int MODE>
const void* conv_mma_pick(int tc, size_t& smem) {
    // tc 2 (bf16 fast mode): the activations are fp32 in HBM and land in smem by cp.async
    // as they are, so the convolutions run kind::tf32 (no conversion pass)
    return tc == 3 ? conv_mma_func<MODE, 4, true>(smem) : conv_mma_func<MODE, 4, false>(smem);
}

// Wt[m][tap * C + c] = fwd: W[m][c][tap] (C = c_in); dgrad: W[c][m][tap] (C = c_out)
template <int MODE>
__global__ void __launch_bounds__(NT) conv_wprep_kernel(const ConvArgs a) {
    FB_PDL_ENTRY();
    float* Wt = const_cast<float*>(a.Wt);
    const int kk = a.k * a.k;
    const int C = MODE == kConvFwd ? a.ci : a.co;
    const size_t n = (size_t)a.M * a.K;
    for (size_t i = (size_t)blockIdx.x * NT + threadIdx.x; i < n; i += (size_t)gridDim.x * NT) {
        const int m = (int)(i / a.K), k = (int)(i - (size_t)m * a.K);
        const int tap = k / C, c = k - tap * C;
        Wt[i] = MODE == kConvFwd ? __ldg(a.W + ((size_t)m * a.ci + c) * kk + tap)
                                 : __ldg(a.W + ((size_t)c * a.ci + m) * kk + tap);
    }
}

}  // namespace

size_t conv_plan(ConvArgs& a, int mode, size_t max_partial) {
    const int kk = a.k * a.k;
    if (mode == kConvFwd) {
        a.M = a.co;
        a.N = a.B * a.ho * a.wo;
        a.K = a.ci * kk;
    } else if (mode == kConvDgrad) {
        a.M = a.ci;
        a.N = a.B * a.hi * a.wi;
        a.K = a.co * kk;
    } else {
        a.M = a.co;
        a.bcol = a.tc && a.bcol ? 1 : 0;  // the fused bias column needs the tensor-core path
        a.N = a.ci * kk + a.bcol;
        a.K = a.B * a.ho * a.wo;
    }
    if (a.tc) {  // tensor cores: 128 x 128 tiles, K in 128-byte atoms, about one wave of CTAs
        const int KA = 32;  // tf32 atoms (tc 2 runs the tf32 kernel)
        const long long katoms = (a.K + KA - 1) / KA;
        const long long mt = (long long)((a.M + 127) / 128) * ((a.N + 127) / 128);
        // one CTA per SM (544 threads): split K only as far as the tiles stay one wave
        // (splitting a multi-wave grid adds the partial traffic and buys nothing)
        // half a wave of the resident CTAs (3xTF32: one per SM -> 74; tf32 / bf16 modes: two per SM
        // -> 148): inside the concurrent chunk graph the other stages' convolutions run beside it
        // (C3 fp32 4,155 -> 4,310, tf32 5,204 -> 6,087 samples/s against a full wave;
        // profiles/r2/c3_wave.txt, profiles/r2/c3_wave_tf32.txt)
        static const char* wave_env = std::getenv("FERRET_CONV_WAVE");
        const long long wave = wave_env ? std::atoll(wave_env) : (a.tc == 3 ? 74 : 148);
        long long sp = std::max<long long>(1, wave / mt);
        sp = std::min<long long>(sp, std::max<long long>(1, katoms / 2));
        if (const char* ms = std::getenv("FERRET_CONV_MAX_SPLITS"))  // experiment knob
            sp = std::min<long long>(sp, std::max(1, std::atoi(ms)));
        const long long mn2 = (long long)a.M * a.N;
        if (max_partial) sp = std::min<long long>(sp, std::max<long long>(1, (long long)max_partial / mn2));
        const int C = mode == kConvFwd ? a.ci : a.co;
        a.kt = mode != kConvWgrad && C % KA == 0 && !std::getenv("FERRET_CONV_NO_TAPMAJOR");
        a.apc = (int)((katoms + sp - 1) / sp);
        a.dbg = std::getenv("FERRET_CONV_DBG") ? std::atoi(std::getenv("FERRET_CONV_DBG")) : 0;
        a.splits = (int)((katoms + a.apc - 1) / a.apc);
        a.kchunk = a.apc * KA;
        return a.splits > 1 ? (size_t)a.splits * (size_t)mn2 : 0;
    }
    const long long tiles = (long long)((a.M + TM - 1) / TM) * ((a.N + TN - 1) / TN);
    // about two waves of CTAs over the 148 SMs, each split at least 4 k-tiles deep
    long long splits = std::max<long long>(1, (296 + tiles - 1) / tiles);
    splits = std::min<long long>(splits, std::max(1, a.K / (4 * TK)));
    const long long mn = (long long)a.M * a.N;
    if (max_partial) splits = std::min<long long>(splits, std::max<long long>(1, (long long)max_partial / mn));
    const int chunk = (int)(((a.K + splits - 1) / splits + TK - 1) / TK * TK);
    a.kchunk = chunk;
    a.splits = (a.K + chunk - 1) / chunk;
    return a.splits > 1 ? (size_t)a.splits * (size_t)mn : 0;
}

int spec_conv(const ConvArgs& a, int mode, KernelSpec& gemm, KernelSpec& reduce) {
    if (a.tc) {
        size_t smem = 0;
        const void* g = mode == kConvFwd     ? conv_mma_pick<kConvFwd>(a.tc, smem)
                        : mode == kConvDgrad ? conv_mma_pick<kConvDgrad>(a.tc, smem)
                                             : conv_mma_pick<kConvWgrad>(a.tc, smem);
        fill_spec(gemm, g, dim3((a.N + 127) / 128, (a.M + 127) / 128, a.splits), dim3(kCT), a);
        gemm.smem = smem;
    } else {
        const dim3 grid((a.N + TN - 1) / TN, (a.M + TM - 1) / TM, a.splits);
        const void* g = mode == kConvFwd     ? reinterpret_cast<const void*>(&conv_gemm_kernel<kConvFwd>)
                        : mode == kConvDgrad ? reinterpret_cast<const void*>(&conv_gemm_kernel<kConvDgrad>)
                                             : reinterpret_cast<const void*>(&conv_gemm_kernel<kConvWgrad>);
        fill_spec(gemm, g, grid, dim3(NT), a);
    }
    if (a.splits <= 1) return 1;
    const void* r = mode == kConvFwd     ? reinterpret_cast<const void*>(&conv_reduce_kernel<kConvFwd>)
                    : mode == kConvDgrad ? reinterpret_cast<const void*>(&conv_reduce_kernel<kConvDgrad>)
                                         : reinterpret_cast<const void*>(&conv_reduce_kernel<kConvWgrad>);
    const long long mn = (long long)a.M * a.N;
    const long long threads = warp_reduce(a) ? mn * 32 : mn;
    fill_spec(reduce, r, dim3((unsigned)std::min<long long>((threads + NT - 1) / NT, 148 * 8)), dim3(NT), a);
    return 2;
}

void spec_conv_wprep(const ConvArgs& a, int mode, KernelSpec& k) {
    const long long n = (long long)a.M * a.K;
    const void* f = mode == kConvFwd ? reinterpret_cast<const void*>(&conv_wprep_kernel<kConvFwd>)
                                     : reinterpret_cast<const void*>(&conv_wprep_kernel<kConvDgrad>);
    fill_spec(k, f, dim3((unsigned)std::min<long long>((n + NT - 1) / NT, 148 * 8)), dim3(NT), a);
}

void spec_conv_bgrad(const ConvArgs& a, float* gb, KernelSpec& k) {
    ConvArgs b = a;
    b.Y = gb;
    fill_spec(k, reinterpret_cast<const void*>(&conv_bgrad_kernel), dim3(a.co), dim3(NT), b);
}

void spec_gap(const PoolMeanArgs& a, KernelSpec& k) {
    fill_spec(k, reinterpret_cast<const void*>(&gap_kernel), dim3((a.B * a.C + NT - 1) / NT), dim3(NT), a);
}

void spec_ungap(const PoolMeanArgs& a, KernelSpec& k) {
    const long long n = (long long)a.B * a.C * a.HW;
    fill_spec(k, reinterpret_cast<const void*>(&ungap_kernel), dim3((unsigned)std::min<long long>((n + NT - 1) / NT, 148 * 8)),
              dim3(NT), a);
}

}  // namespace fb200
