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
// 64 x 64 CTA tiles, K in steps of 16 through shared memory, 4 x 4 fp32
// accumulators per thread (SIMT FFMA: the fp32 parity mode's arithmetic). Grids
// with few tiles split K over blockIdx.z into a partial buffer, reduced in split
// order by a second kernel that also runs the epilogue, so results do not depend
// on scheduling (bitwise reproducible).
#include "kernels.cuh"

#include <algorithm>
#include <cstring>

namespace fb200 {

namespace {

constexpr int TM = 64, TN = 64, TK = 16, NT = 256;

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
        a.Y[(size_t)m * a.N + n] = v;
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

// ordered sum of the K-split partials, then the epilogue
template <int MODE>
__global__ void __launch_bounds__(NT) conv_reduce_kernel(const ConvArgs a) {
    const size_t mn = (size_t)a.M * a.N;
    for (size_t i = (size_t)blockIdx.x * NT + threadIdx.x; i < mn; i += (size_t)gridDim.x * NT) {
        float v = 0.f;
        for (int s = 0; s < a.splits; ++s) v += __ldg(a.partial + (size_t)s * mn + i);
        const int m = (int)(i / a.N), n = (int)(i - (size_t)m * a.N);
        epilogue<MODE>(a, m, n, v);
    }
}

// gb[co] = sum_b sum_pix D[b][co][pix]: one warp per channel, fixed order
// (gb = a.Y)
__global__ void __launch_bounds__(NT) conv_bgrad_kernel(const ConvArgs a) {
    const int warp = (blockIdx.x * NT + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= a.co) return;
    const int hw = a.ho * a.wo;
    float v = 0.f;
    for (int b = 0; b < a.B; ++b) {
        const float* d = a.D + ((size_t)b * a.co + warp) * hw;
        for (int p = lane; p < hw; p += 32) v += __ldg(d + p);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) a.Y[warp] = v;
}

__global__ void __launch_bounds__(NT) gap_kernel(const PoolMeanArgs a) {
    const int i = blockIdx.x * NT + threadIdx.x;
    if (i >= a.B * a.C) return;
    const int b = i / a.C, c = i - b * a.C;
    const float* x = a.X + (a.xidx ? (size_t)__ldg(a.xidx + b) : (size_t)b) * a.C * a.HW + (size_t)c * a.HW;
    float s = 0.f;
    for (int p = 0; p < a.HW; ++p) s += __ldg(x + p);
    a.Y[i] = s / (float)a.HW;
}

__global__ void __launch_bounds__(NT) ungap_kernel(const PoolMeanArgs a) {
    const size_t n = (size_t)a.B * a.C * a.HW;
    for (size_t i = (size_t)blockIdx.x * NT + threadIdx.x; i < n; i += (size_t)gridDim.x * NT) {
        float v = __ldg(a.dY + i / a.HW) / (float)a.HW;
        if (a.mask && !(__ldg(a.mask + i) > 0.f)) v = 0.f;
        a.dX[i] = v;
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
        a.N = a.ci * kk;
        a.K = a.B * a.ho * a.wo;
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
    const dim3 grid((a.N + TN - 1) / TN, (a.M + TM - 1) / TM, a.splits);
    const void* g = mode == kConvFwd     ? reinterpret_cast<const void*>(&conv_gemm_kernel<kConvFwd>)
                    : mode == kConvDgrad ? reinterpret_cast<const void*>(&conv_gemm_kernel<kConvDgrad>)
                                         : reinterpret_cast<const void*>(&conv_gemm_kernel<kConvWgrad>);
    fill_spec(gemm, g, grid, dim3(NT), a);
    if (a.splits <= 1) return 1;
    const void* r = mode == kConvFwd     ? reinterpret_cast<const void*>(&conv_reduce_kernel<kConvFwd>)
                    : mode == kConvDgrad ? reinterpret_cast<const void*>(&conv_reduce_kernel<kConvDgrad>)
                                         : reinterpret_cast<const void*>(&conv_reduce_kernel<kConvWgrad>);
    const long long mn = (long long)a.M * a.N;
    fill_spec(reduce, r, dim3((unsigned)std::min<long long>((mn + NT - 1) / NT, 148 * 8)), dim3(NT), a);
    return 2;
}

void spec_conv_bgrad(const ConvArgs& a, float* gb, KernelSpec& k) {
    ConvArgs b = a;
    b.Y = gb;
    fill_spec(k, reinterpret_cast<const void*>(&conv_bgrad_kernel), dim3((a.co * 32 + NT - 1) / NT), dim3(NT), b);
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
