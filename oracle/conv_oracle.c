/*
 * conv_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of the three operators on
 * the hot path of arXiv 2305.08819 (Dragon-Alpha & cu32): fp32 2-D convolution
 * forward, deconvolution (input gradient) and weight gradient, NHWC activations,
 * filters [OC,FH,FW,IC].
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl
 * reference) may load this library.  It shares no code, header, helper or
 * constant with the CUDA path under paper_2305_08819_b200/csrc/, and the CUDA
 * path never calls it.
 *
 * Sources of the definitions (the paper never writes the formulas; it names the
 * operators and fixes layout / precision):
 *   - PAPER.md:115 (§II "High-performance"): "the matrix-multiply and
 *     convolution\deconvolution (conv\deconv) operators are highly optimized";
 *     last dimension padded to 4x.
 *   - PAPER.md:180 (Table I): activations are [N, H, W, C] (NHWC), float32.
 *   - PAPER.md:42 (Fig. 2): nn.conv3D(false, in, out, k, stride, pad) — one pad
 *     argument, symmetric; no bias.
 *   - SPEC.md:104-132 (backend module): conv2d_forward / backward_data /
 *     backward_filter post-conditions, filter layout [out_c, kh, kw, in_c],
 *     cross-correlation (no kernel flip).
 *   - DESIGN.md "Readings" L1 (floor output size), L5 (dX has the forward input's
 *     extent), L6 (all three overwrite).
 *
 * Arithmetic: every product of two fp32 numbers is exact in double (24+24 < 53
 * significand bits); sums are accumulated in double in the fixed order stated at
 * each function.  OpenMP parallelises over OUTPUT elements only, so every output
 * element is computed by one thread in the same order whatever the thread count.
 */
#include <stddef.h>
#include <stdint.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_OK 0
#define ORACLE_EARG 1

/* Reading L1: OH = floor((IH + 2*ph - FH) / sh) + 1, required >= 1. */
int oracle_out_hw(int IH, int IW, int FH, int FW, int sh, int sw, int ph, int pw,
                  int* OH, int* OW) {
    if (IH < 1 || IW < 1 || FH < 1 || FW < 1 || sh < 1 || sw < 1 || ph < 0 || pw < 0)
        return ORACLE_EARG;
    int nh = IH + 2 * ph - FH, nw = IW + 2 * pw - FW;
    if (nh < 0 || nw < 0) return ORACLE_EARG;
    *OH = nh / sh + 1;
    *OW = nw / sw + 1;
    return ORACLE_OK;
}

/*
 * O1 forward:
 *   Y[n,oh,ow,oc] = sum_{fh<FH} sum_{fw<FW} sum_{ic<IC}
 *                   X[n, oh*sh-ph+fh, ow*sw-pw+fw, ic] * W[oc,fh,fw,ic]
 * with X outside [0,IH)x[0,IW) taken as 0 (zero padding).  Order: fh, fw, ic.
 */
int oracle_conv2d_fwd(const float* X, const float* W, double* Y,
                      int N, int IH, int IW, int IC, int OC, int FH, int FW,
                      int sh, int sw, int ph, int pw) {
    int OH, OW;
    if (N < 1 || IC < 1 || OC < 1) return ORACLE_EARG;
    if (oracle_out_hw(IH, IW, FH, FW, sh, sw, ph, pw, &OH, &OW)) return ORACLE_EARG;
    const long long total = (long long)N * OH * OW * OC;
#pragma omp parallel for schedule(static)
    for (long long e = 0; e < total; ++e) {
        long long r = e;
        const int oc = (int)(r % OC); r /= OC;
        const int ow = (int)(r % OW); r /= OW;
        const int oh = (int)(r % OH); r /= OH;
        const int n = (int)r;
        double acc = 0.0;
        for (int fh = 0; fh < FH; ++fh) {
            const int ih = oh * sh - ph + fh;
            if (ih < 0 || ih >= IH) continue;          /* padding contributes 0 */
            for (int fw = 0; fw < FW; ++fw) {
                const int iw = ow * sw - pw + fw;
                if (iw < 0 || iw >= IW) continue;
                const float* x = X + (((size_t)n * IH + ih) * IW + iw) * IC;
                const float* w = W + (((size_t)oc * FH + fh) * FW + fw) * IC;
                for (int ic = 0; ic < IC; ++ic) acc += (double)x[ic] * (double)w[ic];
            }
        }
        Y[e] = acc;
    }
    return ORACLE_OK;
}

/*
 * O2 deconvolution / input gradient ("full transposed-convolution
 * of dy with w (gradient of conv2d_forward w.r.t. x)"), in
 * gather form, the exact adjoint of O1:
 *   dX[n,ih,iw,ic] = sum_{fh,fw,oc} dY[n,oh,ow,oc] * W[oc,fh,fw,ic]
 *   over the (fh,fw) with ih+ph-fh = oh*sh, iw+pw-fw = ow*sw for integers
 *   0<=oh<OH, 0<=ow<OW.  dX has the forward input's extent (IH,IW) (reading L5);
 *   positions no tap reaches are 0.  Order: fh, fw, oc.
 */
int oracle_conv2d_bwd_data(const float* dY, const float* W, double* dX,
                           int N, int IH, int IW, int IC, int OC, int FH, int FW,
                           int sh, int sw, int ph, int pw) {
    int OH, OW;
    if (N < 1 || IC < 1 || OC < 1) return ORACLE_EARG;
    if (oracle_out_hw(IH, IW, FH, FW, sh, sw, ph, pw, &OH, &OW)) return ORACLE_EARG;
    const long long total = (long long)N * IH * IW * IC;
#pragma omp parallel for schedule(static)
    for (long long e = 0; e < total; ++e) {
        long long r = e;
        const int ic = (int)(r % IC); r /= IC;
        const int iw = (int)(r % IW); r /= IW;
        const int ih = (int)(r % IH); r /= IH;
        const int n = (int)r;
        double acc = 0.0;
        for (int fh = 0; fh < FH; ++fh) {
            const int th = ih + ph - fh;               /* = oh*sh */
            if (th < 0 || th % sh != 0) continue;
            const int oh = th / sh;
            if (oh >= OH) continue;
            for (int fw = 0; fw < FW; ++fw) {
                const int tw = iw + pw - fw;           /* = ow*sw */
                if (tw < 0 || tw % sw != 0) continue;
                const int ow = tw / sw;
                if (ow >= OW) continue;
                const float* dy = dY + (((size_t)n * OH + oh) * OW + ow) * OC;
                for (int oc = 0; oc < OC; ++oc)
                    acc += (double)dy[oc] * (double)W[(((size_t)oc * FH + fh) * FW + fw) * IC + ic];
            }
        }
        dX[e] = acc;
    }
    return ORACLE_OK;
}

/*
 * O3 weight gradient:
 *   dW[oc,fh,fw,ic] = sum_{n,oh,ow} dY[n,oh,ow,oc] * X[n, oh*sh-ph+fh, ow*sw-pw+fw, ic]
 * with out-of-range X = 0.  Order: n, oh, ow.  Overwrites dW (reading L6).
 */
int oracle_conv2d_bwd_filter(const float* X, const float* dY, double* dW,
                             int N, int IH, int IW, int IC, int OC, int FH, int FW,
                             int sh, int sw, int ph, int pw) {
    int OH, OW;
    if (N < 1 || IC < 1 || OC < 1) return ORACLE_EARG;
    if (oracle_out_hw(IH, IW, FH, FW, sh, sw, ph, pw, &OH, &OW)) return ORACLE_EARG;
    const long long total = (long long)OC * FH * FW * IC;
#pragma omp parallel for schedule(static)
    for (long long e = 0; e < total; ++e) {
        long long r = e;
        const int ic = (int)(r % IC); r /= IC;
        const int fw = (int)(r % FW); r /= FW;
        const int fh = (int)(r % FH); r /= FH;
        const int oc = (int)r;
        double acc = 0.0;
        for (int n = 0; n < N; ++n)
            for (int oh = 0; oh < OH; ++oh) {
                const int ih = oh * sh - ph + fh;
                if (ih < 0 || ih >= IH) continue;
                for (int ow = 0; ow < OW; ++ow) {
                    const int iw = ow * sw - pw + fw;
                    if (iw < 0 || iw >= IW) continue;
                    acc += (double)dY[(((size_t)n * OH + oh) * OW + ow) * OC + oc] *
                           (double)X[(((size_t)n * IH + ih) * IW + iw) * IC + ic];
                }
            }
        dW[e] = acc;
    }
    return ORACLE_OK;
}

/*
 * O3 at selected entries only (full-size parity on sampled outputs: "dW parity
 * always uses the full batch"): out[i] = dW[idx[i]] for flat indices into [OC][FH][FW][IC], each
 * computed exactly as oracle_conv2d_bwd_filter computes it (same terms, same n, oh, ow order), so
 * it equals that function's entry bit for bit (pinned in tests/test_oracle_pins.py).
 */
int oracle_conv2d_bwd_filter_at(const float* X, const float* dY, const long long* idx, int nidx, double* out,
                                int N, int IH, int IW, int IC, int OC, int FH, int FW,
                                int sh, int sw, int ph, int pw) {
    int OH, OW;
    if (N < 1 || IC < 1 || OC < 1 || nidx < 0) return ORACLE_EARG;
    if (oracle_out_hw(IH, IW, FH, FW, sh, sw, ph, pw, &OH, &OW)) return ORACLE_EARG;
    const long long total = (long long)OC * FH * FW * IC;
    for (int i = 0; i < nidx; ++i)
        if (idx[i] < 0 || idx[i] >= total) return ORACLE_EARG;
#pragma omp parallel for schedule(dynamic, 1)
    for (int i = 0; i < nidx; ++i) {
        long long r = idx[i];
        const int ic = (int)(r % IC); r /= IC;
        const int fw = (int)(r % FW); r /= FW;
        const int fh = (int)(r % FH); r /= FH;
        const int oc = (int)r;
        double acc = 0.0;
        for (int n = 0; n < N; ++n)
            for (int oh = 0; oh < OH; ++oh) {
                const int ih = oh * sh - ph + fh;
                if (ih < 0 || ih >= IH) continue;
                for (int ow = 0; ow < OW; ++ow) {
                    const int iw = ow * sw - pw + fw;
                    if (iw < 0 || iw >= IW) continue;
                    acc += (double)dY[(((size_t)n * OH + oh) * OW + ow) * OC + oc] *
                           (double)X[(((size_t)n * IH + ih) * IW + iw) * IC + ic];
                }
            }
        out[i] = acc;
    }
    return ORACLE_OK;
}

/* Number of OpenMP threads the oracle will use (for the cpu_baseline "cores"). */
int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void oracle_set_num_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}
