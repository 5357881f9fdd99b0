// smconv.cu — host side of libsmconv: the C ABI of include/smconv.h.
//
// Validation (SPEC.md:332-340 params-check), output-extent algebra
// (reading L1), the per-shape plan ("heuristic table", north_star (c)
// "selected, if feature maps are smaller than a certain threshold"), workspace sizing,
// and kernel launches on the caller's stream.  No allocation, no printing, no exit.
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>

#include "../../include/smconv.h"
#include "../../include/smconv_ext.h"
#include "../../include/smconv_epi.h"
#include "../../include/smconv_mcast.h"
#include "../../include/smgemm.h"
#include "conv_gen.cuh"
#include "conv_strip.cuh"
#include "launch.cuh"

namespace smconv {  // conv_direct.cu
bool direct_supported(int op, int IC, int OC, int FH, int FW, int OW, int sw);
int direct_dw_blocks(int N, int OH);
int direct_launch(int op, const GenParams& g, int blocks, cudaStream_t st, char* err, size_t errlen);
int tma_set_pair(int on);
int tma_get_pair();
bool dws_supported(int op, int IC, int OC, int FH, int FW, int sh, int sw, int OH, int OW);
int dws_splits(int N, int OH, int OW, int* kb_per_split);
int dws_pair_mode();
int dws_hyb_mode();
int dws_launch(int planes, const GenParams& g, int splits, int kb_per_split, cudaStream_t st, char* err,
               size_t errlen);
bool stem_supported(int op, int IC, int OC, int FH, int FW);
int stem_dw_split(long long M, int OC, int* kb_per_cta);
int stem_launch(int op, int planes, const GenParams& g, int splits, int kb_per_split, cudaStream_t st, char* err,
                size_t errlen);
}  // namespace smconv

using namespace smconv;

namespace {

thread_local char g_detail[512] = "";

int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_detail, sizeof g_detail, fmt, ap);
    va_end(ap);
    return code;
}

std::atomic<unsigned long long*> g_trace{nullptr};  // smconv_set_trace (experiments)
std::atomic<int> g_force[3] = {{CONV_VARIANT_AUTO}, {CONV_VARIANT_AUTO}, {CONV_VARIANT_AUTO}};
std::once_flag g_env_once;

void read_env_once() {
    std::call_once(g_env_once, [] {
        const char* e = getenv("SMCONV_FORCE_VARIANT");
        if (!e) return;
        std::string s(e);
        size_t i = 0;
        while (i < s.size()) {
            size_t j = s.find(',', i);
            if (j == std::string::npos) j = s.size();
            std::string item = s.substr(i, j - i);
            int op = -1, var = -1;
            if (sscanf(item.c_str(), "%d:%d", &op, &var) == 2 && op >= 0 && op < 3 && var >= 0 && var <= 5)
                g_force[op].store(var);
            i = j + 1;
        }
    });
}

struct Dims {
    int N, IH, IW, IC, OC, FH, FW, sh, sw, ph, pw, OH, OW;
};

thread_local const char* g_api_name = nullptr;  // the GEMM entry points report their own name

const char* op_name(int op) {
    if (g_api_name) return g_api_name;
    return op == CONV_OP_FWD ? "conv2d_fwd" : op == CONV_OP_BWD_DATA ? "conv2d_bwd_data" : "conv2d_bwd_filter";
}

// The paper's matrix-multiply operators as 1x1 convolutions on a 1x1 map (H = W = 1; the
// "pixels" are the matrix rows), so they run on the same tcgen05 mainloops, plans and epilogues:
//   matMul   C[M,N] = A[M,K] . B[K,N]    = conv2d_bwd_data  (dY = A, W = B as [OC=K][IC=N])
//   matMulT1 C[M,N] = A[K,M]^T . B[K,N]  = conv2d_bwd_filter(X = B [K][N], dY = A [K][M])
//   matMulT2 C[M,N] = A[M,K] . B[N,K]^T  = conv2d_fwd       (X = A [M][K], W = B [OC=N][IC=K])
struct GemmMap {
    int op;
    int dims[11];
};
GemmMap gemm_map(int g, int M, int N, int K) {
    GemmMap m;
    if (g == 0) {
        m.op = CONV_OP_BWD_DATA;
        const int d[11] = {M, 1, 1, N, K, 1, 1, 1, 1, 0, 0};
        memcpy(m.dims, d, sizeof d);
    } else if (g == 1) {
        m.op = CONV_OP_BWD_FILTER;
        const int d[11] = {K, 1, 1, N, M, 1, 1, 1, 1, 0, 0};
        memcpy(m.dims, d, sizeof d);
    } else {
        m.op = CONV_OP_FWD;
        const int d[11] = {M, 1, 1, K, N, 1, 1, 1, 1, 0, 0};
        memcpy(m.dims, d, sizeof d);
    }
    return m;
}
const char* gemm_name(int g) { return g == 0 ? "matMul" : g == 1 ? "matMulT1" : "matMulT2"; }

int check_dims(int op, Dims& d, int math) {
    const char* f = (op >= 0 && op < 3) ? op_name(op) : "conv2d";
    if (op < 0 || op > 2) return fail(CONV_EARG, "%s: unknown op %d", f, op);
    if (math != CONV_MATH_FP32_3XTF32 && math != CONV_MATH_TF32)
        return fail(CONV_EARG, "%s: math=%d is neither CONV_MATH_FP32_3XTF32 (0) nor CONV_MATH_TF32 (1)", f, math);
    const int pos[9] = {d.N, d.IH, d.IW, d.IC, d.OC, d.FH, d.FW, d.sh, d.sw};
    const char* nm[9] = {"N", "IH", "IW", "IC", "OC", "FH", "FW", "sh", "sw"};
    for (int i = 0; i < 9; ++i)
        if (pos[i] < 1) return fail(CONV_EARG, "%s: %s=%d must be >= 1", f, nm[i], pos[i]);
    if (d.ph < 0 || d.pw < 0) return fail(CONV_EARG, "%s: padding (%d,%d) must be >= 0", f, d.ph, d.pw);
    if (conv2d_out_hw(d.IH, d.IW, d.FH, d.FW, d.sh, d.sw, d.ph, d.pw, &d.OH, &d.OW) != CONV_OK)
        return fail(CONV_EARG, "%s: output extent < 1 for IH=%d IW=%d FH=%d FW=%d s=(%d,%d) p=(%d,%d)", f, d.IH,
                    d.IW, d.FH, d.FW, d.sh, d.sw, d.ph, d.pw);
    if (d.IC % 4 || d.OC % 4)
        return fail(CONV_EALIGN, "%s: IC=%d and OC=%d must be multiples of 4 (last dim padded to 4x)", f, d.IC, d.OC);
    const long long lim = 1ll << 31;
    const long long nx = (long long)d.N * d.IH * d.IW * d.IC, ny = (long long)d.N * d.OH * d.OW * d.OC;
    const long long nw = (long long)d.OC * d.FH * d.FW * d.IC;
    if (nx >= lim || ny >= lim || nw >= lim)
        return fail(CONV_EUNSUPPORTED, "%s: tensors must have < 2^31 elements (X %lld, Y %lld, W %lld)", f, nx, ny,
                    nw);
    if (d.FH * d.FW > kMaxTaps) return fail(CONV_EUNSUPPORTED, "%s: FH*FW=%d > %d", f, d.FH * d.FW, kMaxTaps);
    if (d.sh * d.sw > kMaxPhases)
        return fail(CONV_EUNSUPPORTED, "%s: sh*sw=%d > %d stride phases", f, d.sh * d.sw, kMaxPhases);
    if (d.ph > 127 || d.pw > 127) return fail(CONV_EUNSUPPORTED, "%s: padding > 127", f);
    return CONV_OK;
}

bool overlap(const void* a, size_t na, const void* b, size_t nb) {
    const char* x = (const char*)a;
    const char* y = (const char*)b;
    return x < y + nb && y < x + na;
}

// ------------------------------------------------------------------ plans
struct Plan {
    int variant;  // CONV_VARIANT_GENERIC / CONV_VARIANT_TMA
    int BN;
    int planes;
    int splits;
    uint32_t zero_mask;  // dX stride phases with no tap (zero_phases_kernel)
    dim3 grid;
    size_t ws_bytes;
    size_t wx_off, wx_bytes;  // 3xTF32 fwd / dX (TMA, STRIP): bf16 W' plane in the workspace
    size_t wt_off, wt_bytes;  // 3xTF32 dX (TMA, TmaParams::dx_bk): fp32 Wt[IC][T][OC] after it
    long long out_elems;
    GenParams gp;
    TmaParams tp;
    int s2dx;                 // stride-2 3x3 dX as a super-pixel fwd conv (make_plan_s2dx)
    size_t w2_off, w2_bytes;  // its 2x2 filter W2 [(pi, pj, ic)][2][2][OC] in the workspace
    // fused epilogue (smconv_epi.h, csrc/epilogue.cuh)
    int epi;                  // CONV_EPI_*
    int epi_fused;            // 1: in the main kernel's epilogue warps; 0: epi_pass_kernel over the output
    int epi_C, epi_ncols, epi_ngroups, epi_nchunks;
    long long epi_rows;       // pass: output rows (N * H * W)
    size_t epi_part_off, epi_part2_off;  // stats: fp32 partial rows, double chunk sums (workspace)
    int mc_direct;            // fused dW all-reduce: the TMA dW epilogue adds into the multicast address
    int mc_reduce;            //   ... or the split-K reduce kernel does (every other dW plan)
    size_t epi_stage_off;     // pass form of the LEAKY_BWD modes: the conv output is staged here (so that
                              // A may be the output buffer itself: in-place G over A)
};

int pick_bn(int n) {
    if (n <= 32) return 32;
    if (n <= 64) return 64;
    if (n <= 128) return 128;
    return 256;
}

// Largest number of k-blocks (x32 reduction elements) one accumulator chain sums before
// its partial is written out (split-K); bounds TMEM accumulation error.
constexpr int kMaxKbPerChain = 256;
constexpr int kGenMaxKbPerChain3x = 16;  // GENERIC 3xTF32 (no chunked promotion)
// largest cluster split-K (TMA fwd / dX on small maps); SMCONV_CSK=0 turns it off (A/B experiments)
const int g_csk_max = getenv("SMCONV_CSK") ? atoi(getenv("SMCONV_CSK")) : 8;
// make_plan_s2dx: BN cap for the virtual fwd conv it plans (0: none); thread-local, set around one call
thread_local int t_fwd_bn_cap = 0;
// SMCONV_CSK_BN64=1: BN = 64 cluster-split tiles for the smallest maps (see make_plan)
const int g_csk_bn64 = getenv("SMCONV_CSK_BN64") ? atoi(getenv("SMCONV_CSK_BN64")) : 0;
// SMCONV_DX_BK=0: 3xTF32 TMA dX reads the MN-major view of W instead of the transposed plane (A/B)
const int g_dx_bk = getenv("SMCONV_DX_BK") ? atoi(getenv("SMCONV_DX_BK")) : 1;
// SMCONV_ZFILL=0: keep zero_phases_kernel for the 1x1 stride-2 dX (A/B experiments)
const int g_zfill = getenv("SMCONV_ZFILL") ? atoi(getenv("SMCONV_ZFILL")) : 1;
constexpr int kSMs = 148;

void fill_common(GenParams& g, const Dims& d) {
    memset(&g, 0, sizeof g);
    g.N = d.N; g.IH = d.IH; g.IW = d.IW; g.IC = d.IC; g.OC = d.OC; g.FH = d.FH; g.FW = d.FW;
    g.sh = d.sh; g.sw = d.sw; g.ph = d.ph; g.pw = d.pw; g.OH = d.OH; g.OW = d.OW;
    g.fd_N = make_fastdiv(d.N);
    g.fd_OW = make_fastdiv(d.OW);
    g.fd_IC = make_fastdiv(d.IC);
    g.fd_OC = make_fastdiv(d.OC);
    g.fd_FW = make_fastdiv(d.FW);
}

// Valid taps of an output position class — used only to estimate K for split choice.
int est_taps(const Dims& d) {
    // average number of in-bounds taps per output position (fwd)
    long long cnt = 0;
    for (int oh = 0; oh < d.OH; ++oh)
        for (int fh = 0; fh < d.FH; ++fh) cnt += (unsigned)(oh * d.sh - d.ph + fh) < (unsigned)d.IH;
    long long cw = 0;
    for (int ow = 0; ow < d.OW; ++ow)
        for (int fw = 0; fw < d.FW; ++fw) cw += (unsigned)(ow * d.sw - d.pw + fw) < (unsigned)d.IW;
    const double avg = (double)cnt / d.OH * (double)cw / d.OW;
    int t = (int)(avg + 0.999);
    return t < 1 ? 1 : t;
}

// co-resident clusters of S CTAs (1 CTA per SM, ~200 KB smem): 8 GPCs of ~18 SMs hold 15 clusters
// of 8 (ncu launch__cluster_max_active, r02d); a grid of 16 clusters ran in two waves (VGG conv11
// 23.4 us at S = 8 vs 13.8 us at S = 4, r02h), so S is capped to keep one wave
int max_clusters(int S) { return S <= 2 ? 74 : S <= 4 ? 32 : S <= 8 ? 15 : 7; }

// TMA dW on small maps: (BN, split, cluster split) by an estimate in SM cycles.  Per k-block of a
// 128 x BN tile: BN * 2 cycles of TF32 MMA (x3 in 3xTF32); waves of 148 CTAs; a cluster split adds
// the DSMEM reduction of its partial tile (~20 B/cycle/SM, B300_MICROARCH.md) plus two cluster
// barriers; an HBM split adds its partials' write + the reduce kernel's read (6.5 TB/s) and a launch.
const int g_dw_csk = getenv("SMCONV_DW_CSK") ? atoi(getenv("SMCONV_DW_CSK")) : 1;
struct DwChoice { int BN, S, csk; };
DwChoice dw_choose(int planes, int BN0, int m_tiles, int Ngemm, int nkb, int need_prec, int hbm_splits,
                   double out_bytes) {
    const double kSMhz = 1.9e9, kHbm = 6.5e12;
    auto cost = [&](int BN, int S, bool csk) {
        const long long ctas = (long long)m_tiles * ((Ngemm + BN - 1) / BN) * S;
        const double waves = (double)((ctas + kSMs - 1) / kSMs);
        double c = 2500.0 + waves * ((nkb + S - 1) / S) * (2.0 * BN) * (planes == 2 ? 3 : 1);
        if (S > 1 && csk) c += 128.0 * BN * 4 * (S - 1) / S / 20.0 + 3000.0;
        if (S > 1 && !csk) c += (2.0 * S + 1) * out_bytes / kHbm * kSMhz + 6000.0;
        return c;
    };
    const long long hbm_ctas = (long long)m_tiles * ((Ngemm + BN0 - 1) / BN0) * hbm_splits;
    DwChoice best{BN0, hbm_splits, 0};
    double bc = cost(BN0, hbm_splits, false);
    const int bns[2] = {BN0, 128};
    for (int b = 0; b < 2; ++b) {
        const int BN = bns[b];
        if (b == 1 && BN0 <= 128) break;
        const int t2 = m_tiles * ((Ngemm + BN - 1) / BN);
        if (t2 <= kSMs && need_prec <= 1) {  // one chain per tile, no split
            const double c = cost(BN, 1, false);
            if (c < bc) bc = c, best = DwChoice{BN, 1, 0};
        }
        for (int S = 2; S <= g_csk_max && t2 * S <= kSMs && t2 <= max_clusters(S) && 2 * S <= nkb; S *= 2) {
            // measured (r02x, VGG b128 TF32): csk 4 on 72 CTAs lost to the HBM split on 140 (vgg5 dW 28.6 ->
            // 33.2 us); csk 2 on 144 CTAs won over the HBM split 4 (vgg8 29.2 -> 23.0 us)
            if (S < need_prec || 4LL * t2 * S < 3LL * hbm_ctas) continue;
            const double c = cost(BN, S, true);
            if (c < bc) bc = c, best = DwChoice{BN, S, S};
        }
    }
    return best;
}

// SMCONV_HYB_MIN_GFLOP: TMA fwd / dX calls below this much work skip the hybrid form (GenParams::hyb)
std::atomic<double> g_hyb_min_gflop{getenv("SMCONV_HYB_MIN_GFLOP") ? atof(getenv("SMCONV_HYB_MIN_GFLOP")) : 12.0};
// SMCONV_STEM=0: keep the stems on DIRECT / GENERIC (A/B experiments)
const int g_stem = getenv("SMCONV_STEM") ? atoi(getenv("SMCONV_STEM")) : 1;
const long long g_direct_dw_min_rows =
    getenv("SMCONV_DIRECT_DW_MIN_ROWS") ? atoll(getenv("SMCONV_DIRECT_DW_MIN_ROWS")) : 32768;

int make_plan_base(int op, const Dims& d, int math, Plan& pl);
Dims mk(int N, int IH, int IW, int IC, int OC, int FH, int FW, int sh, int sw, int ph, int pw);

// Stride-2 3x3 pad-1 deconvolution (dX of the ResNet stage-entry convs) as ONE stride-1 2x2
// convolution of dY: for the "super-pixel" (i, j) all four stride phases (pi, pj) of dX
// [n, 2i+pi, 2j+pj, :] read dY rows {i, i+1} x columns {j, j+1} only (O2 with ih = 2i+pi:
// pi = 0 takes fh = 1 from oh = i; pi = 1 takes fh = 2 from oh = i and fh = 0 from oh = i+1), so
//   Y2[n, i', j', (pi, pj, ic)] = sum_{a, b, oc} dY[n, i'-1+a, j'-1+b, oc] * W2[(pi, pj, ic), a, b, oc]
// (pad 1, 17x17 outputs for 16x16 dY; i' = i + 1, row / column 0 dropped), with W2 built from W (9 of
// its 16 (tap, phase) blocks non-zero).  dY is read once instead of once per phase and the GEMM is
// N = 4 IC wide with K = 4 OC (full-rate MMAs); the phase walk streamed dY 4x in 128-B rows and
// starved the MMAs (ncu r01r).  The same sums as O2, in a different order.
const int g_s2dx = getenv("SMCONV_S2DX") ? atoi(getenv("SMCONV_S2DX")) : 1;
// SMCONV_S2DX_SKIP=0: issue the all-zero W2 blocks too (A/B experiments)
const int g_s2dx_skip = getenv("SMCONV_S2DX_SKIP") ? atoi(getenv("SMCONV_S2DX_SKIP")) : 1;
// SMCONV_S2DX_BN=64: super-pixel dX with one stride phase (IC columns) per n-tile, so no n-tile issues
// MMAs for another phase's all-zero W2 blocks (25 % fewer MACs at IC = 64), at N = 64 (pair) tiles
const int g_s2dx_bn = getenv("SMCONV_S2DX_BN") ? atoi(getenv("SMCONV_S2DX_BN")) : 0;

int make_plan_s2dx(const Dims& d, int math, Plan& pl) {
    if (!g_s2dx || g_force[CONV_OP_BWD_DATA].load() != CONV_VARIANT_AUTO) return -1;
    if (d.FH != 3 || d.FW != 3 || d.sh != 2 || d.sw != 2 || d.ph != 1 || d.pw != 1) return -1;
    if (d.IH != 2 * d.OH || d.IW != 2 * d.OW || d.IC % 64 || d.OC % 32 || d.N % 32) return -1;
    // Only where the phase walk is starved (r01aa, b4096 3xTF32): dY maps of >= 16x16 positions
    // (l2.0a: 1.71 -> 1.40 ms in the step; TF32 1.13 -> 0.73 ms).  On 8x8 / 4x4 maps dY stays in
    // L2 across the phase passes and the 2x padded-MAC cost of the super-pixel GEMM loses
    // (l3.0a 0.69 -> 1.08 ms, l4.0a 0.51 -> 0.93 ms).
    if (d.OH * d.OW < 256) return -1;
    Dims v = mk(d.N, d.OH, d.OW, d.OC, 4 * d.IC, 2, 2, 1, 1, 1, 1);
    v.OH = d.OH + 1;  // (OH + 2 - 2) / 1 + 1
    v.OW = d.OW + 1;
    t_fwd_bn_cap = (g_s2dx_bn > 0 && d.IC % g_s2dx_bn == 0) ? g_s2dx_bn : 0;
    const int rcb = make_plan_base(CONV_OP_FWD, v, math, pl);
    t_fwd_bn_cap = 0;
    if (rcb) return -1;
    if (pl.variant != CONV_VARIANT_TMA || pl.splits != 1 || pl.zero_mask) return -1;
    pl.s2dx = 1;
    pl.gp.s2dx = 1;
    // per n-tile tap mask (GenParams::s2_tapmask): column (pi, pj, ic) has a non-zero W2 block at tap
    // (a, b) iff (pi == 1 || a == 0) && (pj == 1 || b == 0)
    {
        const int nt = (4 * d.IC + pl.BN - 1) / pl.BN;
        if (nt > 16 || g_s2dx_skip == 0) {
            memset(pl.gp.s2_tapmask, 0xF, sizeof pl.gp.s2_tapmask);
        } else {
            for (int t = 0; t < nt; ++t) {
                uint8_t m = 0;
                const int ph0 = t * pl.BN / d.IC, ph1 = ((t + 1) * pl.BN - 1) / d.IC;
                for (int ph = ph0; ph <= ph1 && ph < 4; ++ph) {
                    const int pi = ph >> 1, pj = ph & 1;
                    for (int a = 0; a < 2; ++a)
                        for (int b = 0; b < 2; ++b)
                            if ((pi == 1 || a == 0) && (pj == 1 || b == 0)) m |= (uint8_t)(1u << (2 * a + b));
                }
                pl.gp.s2_tapmask[t] = m;
            }
        }
    }
    pl.gp.s2_IH = d.IH;
    pl.gp.s2_IW = d.IW;
    pl.gp.s2_IC = d.IC;
    pl.w2_off = (pl.ws_bytes + 1023) & ~(size_t)1023;
    pl.w2_bytes = (size_t)16 * d.IC * d.OC * sizeof(float);
    pl.ws_bytes = pl.w2_off + pl.w2_bytes;
    pl.out_elems = (long long)d.N * d.IH * d.IW * d.IC;
    return 0;
}

// W2[(pi, pj, ic)][a][b][oc] = W[oc][fh(pi, a)][fw(pj, b)][ic], 0 where the phase has no such tap
__global__ void __launch_bounds__(256) w2_build_kernel(const float* __restrict__ W, float* __restrict__ W2, int IC,
                                                       int OC) {
    pdl_trigger();
    pdl_wait();
    const long long n = 16LL * IC * OC;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
        const int oc = (int)(e % OC);
        long long r = e / OC;
        const int b = (int)(r & 1), a = (int)((r >> 1) & 1);
        r >>= 2;
        const int ic = (int)(r % IC);
        const int ph = (int)(r / IC), pi = ph >> 1, pj = ph & 1;
        const int fh = pi == 0 ? (a == 0 ? 1 : -1) : (a == 0 ? 2 : 0);
        const int fw = pj == 0 ? (b == 0 ? 1 : -1) : (b == 0 ? 2 : 0);
        W2[e] = (fh >= 0 && fw >= 0) ? W[(((size_t)oc * 3 + fh) * 3 + fw) * IC + ic] : 0.f;
    }
}

// Fused epilogue (smconv_epi.h): in the conv kernel's epilogue where that kernel writes the final
// values (TMA / STRIP without split-K), else one pass over the output; statistics partial rows of 32
// output rows, summed in fixed order by two small kernels.
void plan_epi(int op, const Dims& d, int epi, Plan& pl) {
    pl.epi = epi;
    if (!epi) return;
    const bool ws_split = pl.splits > 1 && !pl.gp.csk;
    const int C = op == CONV_OP_FWD ? d.OC : d.IC;
    const int oh = op == CONV_OP_FWD ? d.OH : d.IH, ow = op == CONV_OP_FWD ? d.OW : d.IW;
    pl.epi_C = C;
    pl.epi_rows = (long long)d.N * oh * ow;
    pl.epi_fused = (pl.variant == CONV_VARIANT_TMA || pl.variant == CONV_VARIANT_STRIP) && !ws_split && !pl.gp.csk;
    if (pl.epi_fused) {
        if (pl.variant == CONV_VARIANT_STRIP) pl.epi_ngroups = (d.N + 31) / 32 * oh * ow;
        else if (op == CONV_OP_BWD_DATA && !pl.s2dx)  // phase tiles of 128 rows (256 rows for CTA pairs)
            pl.epi_ngroups = pl.gp.phase_tile0[pl.gp.nphase] * (pl.tp.pair ? 8 : 4);
        else pl.epi_ngroups = (pl.gp.M + 127) / 128 * 4;  // fwd, and the super-pixel dX's virtual fwd rows
        pl.epi_ncols = pl.gp.Ngemm;                        // = C, or 4 IC for the super-pixel dX
    } else {
        pl.epi_ngroups = (int)((pl.epi_rows + 31) / 32);
        pl.epi_ncols = C;
        if (epi_reads_a(epi)) {
            pl.epi_stage_off = (pl.ws_bytes + 255) & ~(size_t)255;
            pl.ws_bytes = pl.epi_stage_off + (size_t)pl.epi_rows * C * sizeof(float);
        }
    }
    if (epi_has_stats(epi)) {
        long long nch = 65536 / (2 * pl.epi_ncols);
        if (nch < 1) nch = 1;
        if (nch > pl.epi_ngroups) nch = pl.epi_ngroups;
        pl.epi_nchunks = (int)nch;
        pl.epi_part_off = (pl.ws_bytes + 255) & ~(size_t)255;
        pl.ws_bytes = pl.epi_part_off + (size_t)2 * pl.epi_ngroups * pl.epi_ncols * sizeof(float);
        pl.epi_part2_off = (pl.ws_bytes + 255) & ~(size_t)255;
        pl.ws_bytes = pl.epi_part2_off + (size_t)2 * pl.epi_nchunks * pl.epi_ncols * sizeof(double);
    }
}

// kMcastEpi: plan-cache key of a conv2d_bwd_filter_mcast plan (fused dW + in-switch all-reduce)
constexpr int kMcastEpi = 100;

void plan_mcast(Plan& pl) {
    if (pl.variant == CONV_VARIANT_TMA && pl.splits == 1) {
        pl.mc_direct = 1;
        return;
    }
    pl.mc_reduce = 1;
    if (!(pl.splits > 1 && !pl.gp.csk)) {  // single split: stage the tile in the workspace, reduce kernel adds it
        pl.ws_bytes = (size_t)pl.out_elems * sizeof(float);
        pl.gp.split_stride = pl.out_elems;
    }
}

// split-K reduce form: one warp per output float4 when the output is small (<= 148 x 2048 lanes) and
// the partials many (splitk_reduce_wide_kernel)
bool reduce_wide(long long n4, int splits) { return splits >= 16 && n4 * 32 <= (long long)kSMs * 2048; }

int plan_kernel_count(const Plan& pl) {
    return 1 + ((pl.splits > 1 && !pl.gp.csk) || pl.mc_reduce) + (pl.zero_mask != 0) + (pl.wx_bytes != 0) + (pl.s2dx != 0) +
           (pl.epi && !pl.epi_fused) + 2 * epi_has_stats(pl.epi);
}

int make_plan_uncached(int op, const Dims& d, int math, Plan& pl, int epi) {
    if (op == CONV_OP_BWD_DATA && make_plan_s2dx(d, math, pl) == 0) {
        plan_epi(op, d, epi, pl);
        return CONV_OK;
    }
    const int rc = make_plan_base(op, d, math, pl);
    if (rc == CONV_OK && epi == kMcastEpi) plan_mcast(pl);
    else if (rc == CONV_OK) plan_epi(op, d, epi, pl);
    return rc;
}

// Process-wide plan cache (SURVEY.md §8(b) contract 4): plans hold no pointers, so a plan is a pure
// function of (op, the 11-int conv tuple, math, the forced variant, the CTA-pair switch).  Small-map
// layers run ~10 us kernels; re-deriving the plan (tap tables, split choice) on every call is host
// time on the critical path.  Guarded by a mutex (the library is reentrant across threads/streams).
struct PlanKey {
    int v[16];
    bool operator==(const PlanKey& o) const { return memcmp(v, o.v, sizeof v) == 0; }
};
struct PlanKeyHash {
    size_t operator()(const PlanKey& k) const {
        uint64_t h = 1469598103934665603ull;
        for (int x : k.v) h = (h ^ (uint32_t)x) * 1099511628211ull;
        return (size_t)h;
    }
};
std::mutex g_plan_mu;
std::unordered_map<PlanKey, Plan, PlanKeyHash> g_plans;
constexpr size_t kMaxPlans = 4096;

int make_plan(int op, const Dims& d, int math, Plan& pl, int epi = CONV_EPI_NONE) {
    read_env_once();
    PlanKey k;
    const int v[16] = {op, d.N, d.IH, d.IW, d.IC, d.OC, d.FH, d.FW, d.sh, d.sw, d.ph, d.pw, math,
                       g_force[op].load(), tma_get_pair(), epi};
    memcpy(k.v, v, sizeof v);
    {
        std::lock_guard<std::mutex> lk(g_plan_mu);
        auto it = g_plans.find(k);
        if (it != g_plans.end()) {
            pl = it->second;
            return CONV_OK;
        }
    }
    const int rc = make_plan_uncached(op, d, math, pl, epi);
    if (rc) return rc;  // failures are not cached (their detail string is per call)
    std::lock_guard<std::mutex> lk(g_plan_mu);
    if (g_plans.size() >= kMaxPlans) g_plans.clear();
    g_plans.emplace(k, pl);
    return CONV_OK;
}

int make_plan_base(int op, const Dims& d, int math, Plan& pl) {
    memset(&pl, 0, sizeof pl);
    read_env_once();
    pl.planes = math == CONV_MATH_FP32_3XTF32 ? 2 : 1;
    int forced = g_force[op].load();
    const bool tma_ok = tma_supported(op, d.N, d.IC, d.OC, d.FH, d.FW, d.sh, d.sw);
    pl.variant = forced == CONV_VARIANT_AUTO ? (tma_ok ? CONV_VARIANT_TMA : CONV_VARIANT_GENERIC) : forced;
    if (pl.variant == CONV_VARIANT_TMA && !tma_ok)
        return fail(CONV_EUNSUPPORTED, "%s: TMA variant forced but unsupported for this shape", op_name(op));
    // STRIP serves fwd / dX only (strip_launch treats every non-fwd op as dX)
    if (forced == CONV_VARIANT_STRIP && op == CONV_OP_BWD_FILTER)
        return fail(CONV_EUNSUPPORTED, "%s: STRIP variant forced but it serves fwd / dX only", op_name(op));
    if (op != CONV_OP_BWD_FILTER && (forced == CONV_VARIANT_AUTO || forced == CONV_VARIANT_STRIP)) {
        const int bns = pick_bn(op == CONV_OP_FWD ? d.OC : d.IC);
        const bool strip_ok = strip_supported(op, d.N, d.IC, d.OC, d.FW, d.sh, d.sw, op == CONV_OP_FWD ? d.OW : d.IW,
                                              bns, pl.planes);
        if (strip_ok) pl.variant = CONV_VARIANT_STRIP;
        else if (forced == CONV_VARIANT_STRIP)
            return fail(CONV_EUNSUPPORTED, "%s: STRIP variant forced but unsupported for this shape", op_name(op));
    }
    if (forced == CONV_VARIANT_AUTO || forced == CONV_VARIANT_DIRECT) {
        // few-channel stems: HBM-bound, K = FH*FW*IC tiny -> CUDA-core fp32 direct kernels
        bool direct_ok = direct_supported(op, d.IC, d.OC, d.FH, d.FW, d.OW, d.sw);
        // stem dW with < 32768 (n, oh) rows: the GENERIC tensor-core split-K variant is faster
        // (r01z: VGG b128 60 vs 89 us, GoogLeNet b256 153 vs 417 us, ResNet b512 157 vs 175 us; equal
        // at b1024); at ResNet b4096 (131k rows) DIRECT is (0.92 vs 1.39 ms)
        if (direct_ok && forced == CONV_VARIANT_AUTO && op == CONV_OP_BWD_FILTER && (long long)d.N * d.OH < g_direct_dw_min_rows)
            direct_ok = false;
        if (direct_ok) pl.variant = CONV_VARIANT_DIRECT;
        else if (forced == CONV_VARIANT_DIRECT)
            return fail(CONV_EUNSUPPORTED, "%s: DIRECT variant forced but unsupported for this shape", op_name(op));
    }
    if (forced == CONV_VARIANT_AUTO || forced == CONV_VARIANT_STEM) {
        // few-channel stems on the tensor cores (conv_stem.cu): replaces DIRECT / GENERIC there
        const bool stem_ok = g_stem && stem_supported(op, d.IC, d.OC, d.FH, d.FW) &&
                             (long long)d.N * d.OH * d.OW < (1LL << 31);
        if (stem_ok) pl.variant = CONV_VARIANT_STEM;
        else if (forced == CONV_VARIANT_STEM)
            return fail(CONV_EUNSUPPORTED, "%s: STEM variant forced but unsupported for this shape", op_name(op));
    }
    if (forced == CONV_VARIANT_AUTO || forced == CONV_VARIANT_DWS) {
        const bool dws_ok = dws_supported(op, d.IC, d.OC, d.FH, d.FW, d.sh, d.sw, d.OH, d.OW);
        if (dws_ok) pl.variant = CONV_VARIANT_DWS;
        else if (forced == CONV_VARIANT_DWS)
            return fail(CONV_EUNSUPPORTED, "%s: DWS variant forced but unsupported for this shape", op_name(op));
    }

    // 3xTF32 on the TMA variant promotes chunks into BN/2 fp32 registers per epilogue thread: BN <= 128
    auto bn_for = [&](int n) {
        int b = pick_bn(n);
        if (pl.variant == CONV_VARIANT_TMA && pl.planes == 2 && b > 128) b = 128;
        return b;
    };
    GenParams& g = pl.gp;
    fill_common(g, d);
    long long out_elems;
    int m_tiles, n_tiles, nkb_est;
    if (op == CONV_OP_FWD) {
        g.M = d.N * d.OH * d.OW;
        g.Ngemm = d.OC;
        m_tiles = (g.M + 127) / 128;
        pl.BN = bn_for(g.Ngemm);
        if (t_fwd_bn_cap > 0 && pl.BN > t_fwd_bn_cap) pl.BN = t_fwd_bn_cap;  // make_plan_s2dx
        n_tiles = (g.Ngemm + pl.BN - 1) / pl.BN;
        out_elems = (long long)d.N * d.OH * d.OW * d.OC;
        nkb_est = (est_taps(d) * d.IC + 31) / 32;
    } else if (op == CONV_OP_BWD_DATA) {
        g.Ngemm = d.IC;
        g.nphase = d.sh * d.sw;
        m_tiles = 0;
        for (int rh = 0; rh < d.sh; ++rh)
            for (int rw = 0; rw < d.sw; ++rw) {
                const int ph_i = rh * d.sw + rw;
                const int IHp = (d.IH - rh + d.sh - 1) / d.sh, IWp = (d.IW - rw + d.sw - 1) / d.sw;
                g.phase_rh[ph_i] = rh;
                g.phase_rw[ph_i] = rw;
                g.phase_IHp[ph_i] = IHp;
                g.phase_IWp[ph_i] = IWp;
                g.phase_fd_IWp[ph_i] = make_fastdiv(IWp > 0 ? IWp : 1);
                g.phase_tile0[ph_i] = m_tiles;
                // a phase with no filter tap at all (fh = rh+ph mod sh, fw likewise) is all zeros:
                // no tiles; zero_phases_kernel writes it
                bool th = false, tw = false;
                for (int f = 0; f < d.FH; ++f) th |= ((rh + d.ph - f) % d.sh + d.sh) % d.sh == 0;
                for (int f = 0; f < d.FW; ++f) tw |= ((rw + d.pw - f) % d.sw + d.sw) % d.sw == 0;
                if (th && tw) m_tiles += (IHp * IWp * d.N + 127) / 128;
                else if (pl.variant != CONV_VARIANT_STRIP) pl.zero_mask |= 1u << ph_i;
            }
        g.phase_tile0[g.nphase] = m_tiles;
        pl.BN = bn_for(g.Ngemm);
        n_tiles = (g.Ngemm + pl.BN - 1) / pl.BN;
        out_elems = (long long)d.N * d.IH * d.IW * d.IC;
        const int taps_per_phase = (est_taps(d) + d.sh * d.sw - 1) / (d.sh * d.sw) * 1;
        nkb_est = ((taps_per_phase < 1 ? 1 : taps_per_phase) * d.OC + 31) / 32;
    } else if (pl.variant == CONV_VARIANT_TMA && d.OC <= 64 && d.FH * d.FW * d.IC >= 128 && d.IC % 32 == 0 &&
               d.OC % 32 == 0) {
        // OC <= 64 would leave half of every 128-row MMA empty: transpose the dW GEMM to
        // (tap, IC) rows x OC columns (TMA variant only)
        g.dwt = 1;
        g.M = d.FH * d.FW * d.IC;
        g.Ngemm = d.OC;
        g.P = d.N * d.OH * d.OW;
        m_tiles = (g.M + 127) / 128;
        pl.BN = bn_for(g.Ngemm);
        n_tiles = (g.Ngemm + pl.BN - 1) / pl.BN;
        out_elems = (long long)d.OC * d.FH * d.FW * d.IC;
        nkb_est = (g.P + 31) / 32;
    } else {
        g.M = d.OC;
        g.Ngemm = d.FH * d.FW * d.IC;
        if (pl.variant == CONV_VARIANT_TMA && d.IC % 32) {  // (tap, ic) columns with ic padded to 32
            g.dw_icp = (d.IC + 31) / 32 * 32;
            g.fd_icp = make_fastdiv(g.dw_icp);
            g.Ngemm = d.FH * d.FW * g.dw_icp;
        }
        g.P = d.N * d.OH * d.OW;
        m_tiles = (d.OC + 127) / 128;
        pl.BN = bn_for(g.Ngemm);
        n_tiles = (g.Ngemm + pl.BN - 1) / pl.BN;
        out_elems = (long long)d.OC * d.FH * d.FW * d.IC;
        nkb_est = (g.P + 31) / 32;
    }
    if (pl.variant == CONV_VARIANT_TMA && op != CONV_OP_BWD_FILTER) {
        // per-phase tap tables (GenParams::tf_*): fwd -> all rows/columns, offset = filter index;
        // dx phase (rh, rw) -> filter rows fh with (rh + ph - fh) % sh == 0, offset (rh + ph - fh) / sh
        const int nph = op == CONV_OP_FWD ? 1 : g.nphase;
        for (int k = 0; k < nph; ++k) {
            for (int dim = 0; dim < 2; ++dim) {
                const int F = dim == 0 ? d.FH : d.FW, S = dim == 0 ? d.sh : d.sw, P = dim == 0 ? d.ph : d.pw;
                const int r = op == CONV_OP_FWD ? 0 : (dim == 0 ? g.phase_rh[k] : g.phase_rw[k]);
                int n = 0;
                for (int f = 0; f < F; ++f) {
                    int off = f;
                    if (op == CONV_OP_BWD_DATA) {
                        const int t = r + P - f;
                        if (((t % S) + S) % S != 0) continue;
                        off = t / S;
                    }
                    g.tf_f[k][dim][n] = (int8_t)f;
                    g.tf_off[k][dim][n] = (int16_t)off;
                    ++n;
                }
                g.tf_n[k][dim] = (int8_t)n;
            }
        }
    }
    const int tiles = m_tiles * n_tiles;
    int splits = 1;
    if (pl.variant == CONV_VARIANT_STRIP) {
        // strip tiles (32 images x 4R positions) are plentiful: no split-K
    } else if (pl.variant == CONV_VARIANT_DIRECT) {
        // fwd: one block per output row; dW: per-block partials over (n, oh) rows, fixed-order sum
        if (op == CONV_OP_BWD_FILTER) splits = direct_dw_blocks(d.N, d.OH);
    } else if (pl.variant == CONV_VARIANT_DWS) {
        splits = dws_splits(d.N, d.OH, d.OW, &g.kb_per_split);
    } else if (pl.variant == CONV_VARIANT_STEM) {
        // fwd: persistent CTAs over 128-pixel tiles; dW: per-CTA pixel ranges -> fixed-order partial sum
        if (op == CONV_OP_BWD_FILTER) splits = stem_dw_split((long long)d.N * d.OH * d.OW, d.OC, &g.kb_per_split);
    } else if (op == CONV_OP_BWD_FILTER) {
        // GENERIC accumulates its whole chain in TMEM (no chunked promotion) and tcgen05 adds by
        // truncation, so its 3xTF32 chains are capped at 16 k-blocks (512 products): GoogLeNet b256
        // stem dW with 111-k-block chains measured 1.77e-5 normwise (r02a); a numpy model of the
        // truncating chain gives 1.1e-5 / 4.8e-6 / 3.1e-6 at 1024 / 512 / 256 products (K = 262144)
        const int max_chain = (pl.variant == CONV_VARIANT_GENERIC && pl.planes == 2) ? kGenMaxKbPerChain3x
                                                                                     : kMaxKbPerChain;
        const int need_prec = (nkb_est + max_chain - 1) / max_chain;
        int fill = kSMs / tiles;
        if (fill < 1) fill = 1;
        splits = need_prec > fill ? need_prec : fill;
        if (splits > nkb_est) splits = nkb_est;
        if (splits < 1) splits = 1;
        if (pl.variant == CONV_VARIANT_TMA && !g.dwt && splits > 1 && g_dw_csk) {
            // small maps (VGG b128 8x8 .. 2x2): the HBM split-K above writes splits x |dW| of partials and
            // needs a reduce kernel (vgg11 TF32: 2 x 9.4 MB, 28 us for a 1 GFLOP call).  Pick BN and a
            // cluster split (csk: partials reduced through DSMEM in fixed rank order inside the kernel)
            // by a cycle estimate; keep the HBM split when it is cheaper (b4096-sized K)
            const DwChoice c = dw_choose(pl.planes, pl.BN, m_tiles, g.Ngemm, nkb_est, need_prec, splits,
                                         (double)out_elems * 4);
            pl.BN = c.BN;
            n_tiles = (g.Ngemm + pl.BN - 1) / pl.BN;
            splits = c.S;
            g.csk = c.csk;
        }
        g.kb_per_split = (nkb_est + splits - 1) / splits;
        splits = (nkb_est + g.kb_per_split - 1) / g.kb_per_split;
        if (g.csk) splits = g.csk;  // a cluster has exactly csk CTAs (a split past the end sums nothing)
    } else if (tiles < kSMs && pl.variant == CONV_VARIANT_TMA && g_csk_max >= 2) {
        // small maps (VGG 8x8 .. 2x2 at batch 128): split K inside a cluster and reduce the partial
        // tiles through distributed shared memory (one launch; no HBM workspace, no reduce kernel).
        // S = a power of two <= g_csk_max (8: two clusters per GPC), >= 2 k-blocks per split, and at
        // most ~128 CTAs (a cluster of 8 needs 8 free SMs of one GPC).  TF32 tiles of BN = 256 leave
        // too few tiles to fill the machine at S <= 8: use BN = 128 there.
        if (pl.planes == 1 && pl.BN == 256 && tiles * g_csk_max < 120) {
            pl.BN = 128;
            n_tiles = (g.Ngemm + pl.BN - 1) / pl.BN;
        }
        int t2 = m_tiles * n_tiles;
        // S capped by max_clusters (one wave of co-resident clusters)
        auto pick_s = [&](int tt) {
            int S_ = 1;
            for (int S2 = 2; S2 <= g_csk_max && tt * S2 <= kSMs && tt <= max_clusters(S2) && 2 * S2 <= nkb_est; S2 *= 2)
                S_ = S2;
            return S_;
        };
        int S = pick_s(t2);
        // SMCONV_CSK_BN64: while the cluster split fills at most half of the SMs (2x2 maps at batch 128: 16
        // tiles x 4 = 64 CTAs), halve BN (down to 64): twice the CTAs with the same split
        while (g_csk_bn64 && pl.BN >= 128 && t2 * S <= kSMs / 2 && g.Ngemm % (pl.BN / 2) == 0) {
            const int bh = pl.BN / 2;
            const int th = m_tiles * ((g.Ngemm + bh - 1) / bh);
            const int Sh = pick_s(th);
            if (Sh < 2 || th * Sh <= t2 * S) break;
            pl.BN = bh;
            n_tiles = (g.Ngemm + bh - 1) / bh;
            t2 = th;
            S = Sh;
        }
        if (S >= 2) {
            splits = S;
            g.csk = S;
        } else if (t2 < kSMs) {
            splits = kSMs / t2;
            const int maxs = nkb_est / 4 > 1 ? nkb_est / 4 : 1;
            if (splits > maxs) splits = maxs;
            if (splits < 1) splits = 1;
        }
    } else if (tiles < kSMs) {
        splits = kSMs / tiles;
        const int maxs = nkb_est / 4 > 1 ? nkb_est / 4 : 1;
        if (splits > maxs) splits = maxs;
        if (splits < 1) splits = 1;
    }
    if (pl.variant == CONV_VARIANT_GENERIC && pl.planes == 2 && op != CONV_OP_BWD_FILTER) {
        // the same chain cap for GENERIC fwd / dX (worst-case tile: every tap valid)
        const int srcC = op == CONV_OP_FWD ? d.IC : d.OC;
        const int kb_max = (d.FH * d.FW * srcC + 31) / 32;
        const int need = (kb_max + kGenMaxKbPerChain3x - 1) / kGenMaxKbPerChain3x;
        if (splits < need) splits = need;
    }
    g.splits = splits;
    pl.splits = splits;
    pl.out_elems = out_elems;
    const bool ws_split = splits > 1 && !g.csk;  // cluster split-K needs no HBM partials
    pl.ws_bytes = ws_split ? (size_t)splits * out_elems * sizeof(float) : 0;
    g.split_stride = ws_split ? out_elems : 0;
    pl.wx_off = pl.wx_bytes = 0;
    // TMA fwd / dX in 3xTF32: the hybrid form (W' plane + one bf16 cross-term MMA) costs a wx_prep launch
    // per call; below g_hyb_min_gflop of valid-tap work the call runs three TF32 MMAs with b_lo split in
    // the kernel instead (GenParams::hyb)
    g.hyb = 1;
    if (pl.variant == CONV_VARIANT_TMA && pl.planes == 2 && op != CONV_OP_BWD_FILTER &&
        2.0 * (double)out_elems * est_taps(d) * (op == CONV_OP_FWD ? d.IC : d.OC) < g_hyb_min_gflop.load() * 1e9)
        g.hyb = 0;
    if (pl.planes == 2 && op != CONV_OP_BWD_FILTER && g.hyb &&
        (pl.variant == CONV_VARIANT_TMA || pl.variant == CONV_VARIANT_STRIP)) {
        // W' = [bf16(w_lo) | bf16(w)] per (tap, GEMM column, 32-k block): 4 bytes per weight
        pl.wx_off = (pl.ws_bytes + 1023) & ~(size_t)1023;
        const int Kp = ((op == CONV_OP_FWD ? d.IC : d.OC) + 31) / 32 * 32;  // reduction channels padded to 32
        pl.wx_bytes = (size_t)d.FH * d.FW * (op == CONV_OP_FWD ? d.OC : d.IC) * Kp * 4;
        pl.ws_bytes = pl.wx_off + pl.wx_bytes;
        // dX: the same launch also writes the K-major transposed filter (TmaParams::dx_bk), so the
        // TF32 MMA reads B like the fwd does (the MN-major 32-B-atom B made 3xTF32 dX 9-13 % slower
        // than fwd on the same shape, r02bc; TF32 dX, which reads the MN-major view, runs at fwd speed)
        pl.wt_off = pl.wt_bytes = 0;
        if (op == CONV_OP_BWD_DATA && pl.variant == CONV_VARIANT_TMA && g_dx_bk) {
            pl.wt_off = (pl.ws_bytes + 1023) & ~(size_t)1023;
            pl.wt_bytes = (size_t)d.FH * d.FW * d.OC * d.IC * 4;
            pl.ws_bytes = pl.wt_off + pl.wt_bytes;
        }
    }
    pl.grid = dim3(m_tiles, n_tiles, splits);
    if (pl.variant == CONV_VARIANT_TMA) {
        int rc = tma_make_plan(op, g, pl.BN, pl.planes, pl.tp, pl.grid, g_detail, sizeof g_detail);
        if (rc) return rc;
        pl.tp.dx_bk = pl.wt_bytes ? 1 : 0;
        // 1x1 stride-2 dX (ResNet shortcuts): only phase (0, 0) has a tap; the row-coalesced epilogue
        // writes the three empty phases' zeros beside each of its rows (one pass over dX instead of the
        // conv + a zero_phases_kernel pass that ran at ~3.5 TB/s, ncu r02bb)
        if (op == CONV_OP_BWD_DATA && g_zfill && pl.zero_mask == 0xEu && d.sh == 2 && d.sw == 2 && d.IH % 2 == 0 &&
            d.IW % 2 == 0 && splits == 1 && !g.csk && pl.tp.coalesce && tma_epw(op, pl.BN, pl.planes, pl.tp.pair) > 0) {
            pl.tp.zf1 = d.IC;
            pl.tp.zf2 = (long long)d.IW * d.IC;
            pl.zero_mask = 0;
        }
    }
    return CONV_OK;
}

// ------------------------------------------------------------------ launches
template <int OP, int BN, int PLANES>
int launch_gen_t(const GenParams& g, dim3 grid, cudaStream_t st) {
    using C = GenCfg<OP, BN, PLANES>;
    static std::atomic<unsigned long long> attr_done{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ull << (dev & 63);
    if (!(attr_done.load() & bit)) {
        if (cudaFuncSetAttribute(conv_gen_kernel<OP, BN, PLANES>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 C::SMEM_BYTES) != cudaSuccess)
            return fail(CONV_ECUDA, "cudaFuncSetAttribute(smem=%d): %s", C::SMEM_BYTES,
                        cudaGetErrorString(cudaGetLastError()));
        attr_done.fetch_or(bit);
    }
    if (launch_k(conv_gen_kernel<OP, BN, PLANES>, grid, dim3(C::NTHREADS), C::SMEM_BYTES, st, 1, g) != cudaSuccess)
        return fail(CONV_ECUDA, "cudaLaunchKernelEx(generic): %s", cudaGetErrorString(cudaGetLastError()));
    return CONV_OK;
}

template <int OP, int PLANES>
int launch_gen_bn(int BN, const GenParams& g, dim3 grid, cudaStream_t st) {
    switch (BN) {
        case 32: return launch_gen_t<OP, 32, PLANES>(g, grid, st);
        case 64: return launch_gen_t<OP, 64, PLANES>(g, grid, st);
        case 128: return launch_gen_t<OP, 128, PLANES>(g, grid, st);
        default: return launch_gen_t<OP, 256, PLANES>(g, grid, st);
    }
}

template <int OP>
int launch_gen_op(const Plan& pl, const GenParams& g, cudaStream_t st) {
    return pl.planes == 2 ? launch_gen_bn<OP, 2>(pl.BN, g, pl.grid, st) : launch_gen_bn<OP, 1>(pl.BN, g, pl.grid, st);
}

// W' for the 3xTF32 cross terms (common.cuh "3xTF32 operand split"): row (tap, n, cb) of 64 bf16 =
// [bf16(w_lo) for k = 32cb..32cb+31 | bf16(w) for the same k], w_lo = w - trunc_tf32(w); the GEMM
// column n / reduction index k are (oc, ic) for fwd and (ic, oc) for dX.  One thread per row.
__global__ void __launch_bounds__(256) wx_prep_kernel(const float* __restrict__ W, uint4* __restrict__ Wx, int OC,
                                                      int IC, int T, int dx, float* __restrict__ Wt) {
    pdl_trigger();
    pdl_wait();
    // Kc need not be a multiple of 32 (GoogLeNet 16/24/48/112/...-channel layers): the last block's
    // k >= Kc entries are zero, like the TMA's out-of-bounds fill of the matching A columns
    const int Nn = dx ? IC : OC, Kc = dx ? OC : IC, CB = (Kc + 31) / 32;
    const long long rows = (long long)T * Nn * CB;
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < rows; r += (long long)gridDim.x * blockDim.x) {
        int tap, n, cb;
        if (dx) {  // n fastest across threads: the strided W reads coalesce
            n = (int)(r % Nn);
            const long long q = r / Nn;
            cb = (int)(q % CB);
            tap = (int)(q / CB);
        } else {  // cb fastest: each thread reads 128 contiguous bytes
            cb = (int)(r % CB);
            const long long q = r / CB;
            n = (int)(q % Nn);
            tap = (int)(q / Nn);
        }
        uint32_t lo[16], hi[16];
        float wv[32];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            float w0 = 0.f, w1 = 0.f;
            const int k = 32 * cb + 2 * i;  // Kc % 4 == 0: k and k + 1 are both in range or both out
            if (k < Kc) {
                if (dx) {
                    w0 = W[((size_t)k * T + tap) * IC + n];
                    w1 = W[((size_t)(k + 1) * T + tap) * IC + n];
                } else {
                    const float2 v = *reinterpret_cast<const float2*>(W + ((size_t)n * T + tap) * IC + k);
                    w0 = v.x;
                    w1 = v.y;
                }
            }
            wv[2 * i] = w0;
            wv[2 * i + 1] = w1;
            lo[i] = pack_bf16x2(w0 - __uint_as_float(__float_as_uint(w0) & 0xFFFFE000u),
                                w1 - __uint_as_float(__float_as_uint(w1) & 0xFFFFE000u));
            hi[i] = pack_bf16x2(w0, w1);
        }
        if (Wt) {  // dX: Wt[ic = n][tap][oc = k] for this row's 32 k (Kc % 4 == 0: whole float4s in range)
            float* t = Wt + ((size_t)n * T + tap) * Kc + 32 * cb;
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (32 * cb + 4 * q < Kc)
                    *reinterpret_cast<float4*>(t + 4 * q) = make_float4(wv[4 * q], wv[4 * q + 1], wv[4 * q + 2], wv[4 * q + 3]);
        }
        uint4* o = Wx + (((size_t)tap * Nn + n) * CB + cb) * 8;
#pragma unroll
        for (int i = 0; i < 4; ++i) o[i] = make_uint4(lo[4 * i], lo[4 * i + 1], lo[4 * i + 2], lo[4 * i + 3]);
#pragma unroll
        for (int i = 0; i < 4; ++i) o[4 + i] = make_uint4(hi[4 * i], hi[4 * i + 1], hi[4 * i + 2], hi[4 * i + 3]);
    }
}

struct EpiCall {
    int mode;
    float k;
    const float* A;  // LEAKY_BWD*: activation
    double* stats;   // stats modes: [2][C]
};
constexpr EpiCall kMcastCall{kMcastEpi, 0.f, nullptr, nullptr};

// after the main kernel (and split-K reduce / zero fill): the pass form of the epilogue, then the
// fixed-order statistics reduction.  `conv_out` is where the conv wrote (the staging buffer in the pass
// form of the LEAKY_BWD modes), `out` the caller's output.
int finish_epi(int op, const Plan& pl, const float* conv_out, float* out, void* ws, const EpiCall& ec,
               cudaStream_t st) {
    if (!pl.epi) return CONV_OK;
    EpiArgs ea;
    ea.mode = pl.epi;
    ea.k = ec.k;
    ea.A = ec.A;
    ea.part = epi_has_stats(pl.epi) ? (float*)((char*)ws + pl.epi_part_off) : nullptr;
    ea.ngroups = pl.epi_ngroups;
    ea.ncols = pl.epi_ncols;
    if (!pl.epi_fused) {
        const long long items = (long long)pl.epi_ngroups * ((pl.epi_C + 15) / 16);
        const int blocks = (int)((items + 7) / 8 < kSMs * 8 ? (items + 7) / 8 : kSMs * 8);
        launch_k(epi_pass_kernel<0>, dim3(blocks), dim3(256), 0, st, 1, conv_out, out, pl.epi_rows, pl.epi_C, ea);
    }
    if (epi_has_stats(pl.epi)) {
        double* part2 = (double*)((char*)ws + pl.epi_part2_off);
        const long long n1 = 2LL * pl.epi_nchunks * pl.epi_ncols;
        const int b1 = (int)((n1 + 255) / 256 < kSMs * 8 ? (n1 + 255) / 256 : kSMs * 8);
        launch_k(epi_stats_stage1<0>, dim3(b1), dim3(256), 0, st, 1, (const float*)ea.part, part2, pl.epi_ngroups,
                 pl.epi_ncols, pl.epi_nchunks);
        const int b2 = (2 * pl.epi_C + 255) / 256;
        launch_k(epi_stats_stage2<0>, dim3(b2), dim3(256), 0, st, 1, (const double*)part2, ec.stats, pl.epi_ncols,
                 pl.epi_nchunks, pl.epi_C);
    }
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(CONV_ECUDA, "%s: epilogue launch failed: %s", op_name(op), cudaGetErrorString(e));
    return CONV_OK;
}

int run(int op, const float* A, const float* B, float* out, const Dims& d, int math, void* ws, size_t ws_bytes,
        conv_stream_t stream_, const EpiCall& ec) {
    cudaStream_t st = (cudaStream_t)stream_;
    Plan pl;
    int rc = make_plan(op, d, math, pl, ec.mode);
    if (rc) return rc;
    if (pl.ws_bytes > 0 && (ws == nullptr || ws_bytes < pl.ws_bytes))
        return fail(CONV_EWORKSPACE, "%s: workspace %zu bytes at %p, need %zu (conv2d_workspace_bytes)", op_name(op),
                    ws_bytes, ws, pl.ws_bytes);
    if (pl.ws_bytes > 0 && ((uintptr_t)ws & 15)) return fail(CONV_EALIGN, "%s: workspace not 16-B aligned", op_name(op));
    pdl_this_call() = pdl_mode() == 2 || (pdl_mode() == 1 && pl.planes == 1);  // launch.cuh
    GenParams g = pl.gp;
    g.A = A;
    g.B = B;
    const bool ws_split = (pl.splits > 1 && !pl.gp.csk) || pl.mc_reduce;
    g.out = ws_split ? (float*)ws : out;
    g.Bx = nullptr;
    g.Bt = nullptr;
    g.mc_out = pl.mc_direct ? out : nullptr;  // `out` is the multicast address in the mcast plans
    g.trace = g_trace.load();
    // pass form of the LEAKY_BWD modes: the conv (and its reduce / zero fill) write the staging buffer
    float* conv_out = (pl.epi && !pl.epi_fused && epi_reads_a(pl.epi)) ? (float*)((char*)ws + pl.epi_stage_off) : out;
    if (!ws_split) g.out = conv_out;
    memset(&g.epi, 0, sizeof g.epi);
    if (pl.epi && pl.epi_fused) {
        g.epi.mode = pl.epi;
        g.epi.k = ec.k;
        g.epi.A = ec.A;
        g.epi.part = epi_has_stats(pl.epi) ? (float*)((char*)ws + pl.epi_part_off) : nullptr;
        g.epi.ngroups = pl.epi_ngroups;
        g.epi.ncols = pl.epi_ncols;
    }
    // A launch error is detected with cudaGetLastError() after each launch; an error the caller left
    // pending would be misattributed (and consumed) there, so refuse to enqueue and leave it in place.
    {
        const cudaError_t pend = cudaPeekAtLastError();
        if (pend != cudaSuccess)
            return fail(CONV_ECUDA, "%s: a CUDA error is pending from before this call (%s); not cleared, nothing "
                        "enqueued", op_name(op), cudaGetErrorString(pend));
    }
    if (pl.s2dx) {  // super-pixel stride-2 dX: the virtual fwd conv's filter W2, then its W' plane
        float* w2 = (float*)((char*)ws + pl.w2_off);
        const long long n = 16LL * d.IC * d.OC;
        const int blocks = (int)((n + 255) / 256 < kSMs * 8 ? (n + 255) / 256 : kSMs * 8);
        launch_k(w2_build_kernel, dim3(blocks), dim3(256), 0, st, 1, B, w2, d.IC, d.OC);
        g.B = w2;
        if (pl.wx_bytes) {
            g.Bx = (char*)ws + pl.wx_off;
            const long long rows = 4LL * d.OC * 4 * d.IC / 32;
            const int bl = (int)((rows + 255) / 256 < kSMs * 4 ? (rows + 255) / 256 : kSMs * 4);
            launch_k(wx_prep_kernel, dim3(bl), dim3(256), 0, st, 1, (const float*)w2, (uint4*)g.Bx, 4 * d.IC, d.OC, 4, 0,
                     (float*)nullptr);
        }
        TmaParams tp = pl.tp;
        rc = tma_launch(CONV_OP_FWD, pl.BN, pl.planes, g, tp, pl.grid, st, g_detail, sizeof g_detail);
        if (rc) return rc;
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return fail(CONV_ECUDA, "%s: s2dx launch failed: %s", op_name(op), cudaGetErrorString(e));
        rc = finish_epi(op, pl, conv_out, out, ws, ec, st);
        if (rc) return rc;
        g_detail[0] = 0;
        return CONV_OK;
    }
    if (pl.wx_bytes) {
        g.Bx = (char*)ws + pl.wx_off;
        g.Bt = pl.wt_bytes ? (const float*)((char*)ws + pl.wt_off) : nullptr;
        const long long rows = (long long)pl.wx_bytes / 128;  // one 64-bf16 row per (tap, column, 32-k block)
        const int blocks = (int)((rows + 255) / 256 < kSMs * 4 ? (rows + 255) / 256 : kSMs * 4);
        launch_k(wx_prep_kernel, dim3(blocks), dim3(256), 0, st, 1, B, (uint4*)g.Bx, d.OC, d.IC, d.FH * d.FW,
                 (int)(op == CONV_OP_BWD_DATA), (float*)g.Bt);
    }
    if (pl.variant == CONV_VARIANT_DIRECT) {
        rc = direct_launch(op, g, pl.splits, st, g_detail, sizeof g_detail);
    } else if (pl.variant == CONV_VARIANT_STRIP) {
        rc = strip_launch(op, pl.BN, pl.planes, g, st, g_detail, sizeof g_detail);
    } else if (pl.variant == CONV_VARIANT_STEM) {
        rc = stem_launch(op, pl.planes, g, pl.splits, g.kb_per_split, st, g_detail, sizeof g_detail);
    } else if (pl.variant == CONV_VARIANT_DWS) {
        rc = dws_launch(pl.planes, g, pl.splits, g.kb_per_split, st, g_detail, sizeof g_detail);
    } else if (pl.variant == CONV_VARIANT_TMA) {
        TmaParams tp = pl.tp;
        rc = tma_launch(op, pl.BN, pl.planes, g, tp, pl.grid, st, g_detail, sizeof g_detail);
    } else if (op == CONV_OP_FWD) {
        rc = launch_gen_op<OP_FWD>(pl, g, st);
    } else if (op == CONV_OP_BWD_DATA) {
        rc = launch_gen_op<OP_DX>(pl, g, st);
    } else {
        rc = launch_gen_op<OP_DW>(pl, g, st);
    }
    if (rc) return rc;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(CONV_ECUDA, "%s: kernel launch failed: %s", op_name(op), cudaGetErrorString(e));
    if (ws_split) {
        const long long n4 = pl.out_elems / 4;
        const int nsp = pl.gp.csk ? 1 : pl.splits;
        if (reduce_wide(n4, nsp)) {  // many partials of a small output: one warp per float4
            const int blocks = (int)((n4 * 32 + 255) / 256);
            launch_k(splitk_reduce_wide_kernel<0>, dim3(blocks), dim3(256), 0, st, 1, (const float4*)ws,
                     (float4*)conv_out, n4, nsp, n4, pl.mc_reduce ? out : (float*)nullptr);
        } else {
            int blocks = (int)((n4 + 255) / 256);
            if (blocks > kSMs * 8) blocks = kSMs * 8;
            launch_k(splitk_reduce_kernel<0>, dim3(blocks), dim3(256), 0, st, 1, (const float4*)ws, (float4*)conv_out,
                     n4, nsp, n4, pl.mc_reduce ? out : (float*)nullptr);
        }
        e = cudaGetLastError();
        if (e != cudaSuccess) return fail(CONV_ECUDA, "%s: reduce launch failed: %s", op_name(op), cudaGetErrorString(e));
    }
    if (pl.zero_mask) {  // after the reduce: its workspace never held the empty phases
        const long long rows = (long long)d.N * d.IH;
        const int blocks = (int)(rows < kSMs * 8 ? rows : kSMs * 8);
        launch_k(zero_phases_kernel<0>, dim3(blocks), dim3(256), 0, st, 1, (float4*)conv_out, (long long)d.N * d.IH,
                 d.IC / 4, d.IH, d.IW, d.sh, d.sw,
                                                      pl.zero_mask);
        e = cudaGetLastError();
        if (e != cudaSuccess) return fail(CONV_ECUDA, "%s: zero-fill launch failed: %s", op_name(op), cudaGetErrorString(e));
    }
    rc = finish_epi(op, pl, conv_out, out, ws, ec, st);
    if (rc) return rc;
    g_detail[0] = 0;
    return CONV_OK;
}

int entry(int op, const float* in0, const float* in1, float* out, Dims d, int math, void* ws, size_t ws_bytes,
          conv_stream_t st, const EpiCall& ec = EpiCall{0, 0.f, nullptr, nullptr}) {
    int rc = check_dims(op, d, math);
    if (rc) return rc;
    const char* f = op_name(op);
    if (!in0 || !in1 || !out) return fail(CONV_EARG, "%s: NULL tensor pointer", f);
    if (((uintptr_t)in0 | (uintptr_t)in1 | (uintptr_t)out) & 15)
        return fail(CONV_EALIGN, "%s: tensor pointers must be 16-byte aligned", f);
    const size_t bx = (size_t)d.N * d.IH * d.IW * d.IC * 4, by = (size_t)d.N * d.OH * d.OW * d.OC * 4,
                 bw = (size_t)d.OC * d.FH * d.FW * d.IC * 4;
    size_t b0, b1, bo;
    if (op == CONV_OP_FWD) { b0 = bx; b1 = bw; bo = by; }
    else if (op == CONV_OP_BWD_DATA) { b0 = by; b1 = bw; bo = bx; }
    else { b0 = bx; b1 = by; bo = bw; }
    if (overlap(out, bo, in0, b0) || overlap(out, bo, in1, b1))
        return fail(CONV_EALIAS, "%s: output buffer overlaps an input buffer", f);
    if (ws && (overlap(ws, ws_bytes, in0, b0) || overlap(ws, ws_bytes, in1, b1) || overlap(ws, ws_bytes, out, bo)))
        return fail(CONV_EALIAS, "%s: workspace overlaps a tensor", f);
    if (ec.mode && ec.mode != kMcastEpi) {  // fused-epilogue arguments (smconv_epi.h)
        const bool fwd_ok = op == CONV_OP_FWD && (ec.mode == CONV_EPI_BN_STATS || ec.mode == CONV_EPI_LEAKY);
        const bool dx_ok = op == CONV_OP_BWD_DATA && (ec.mode == CONV_EPI_LEAKY_BWD || ec.mode == CONV_EPI_LEAKY_BWD_STATS);
        if (!fwd_ok && !dx_ok) return fail(CONV_EARG, "%s: epilogue %d is not defined for this op", f, ec.mode);
        if ((ec.mode == CONV_EPI_LEAKY || epi_reads_a(ec.mode)) && !(ec.k > 0.f && ec.k < 3.0e38f))
            return fail(CONV_EARG, "%s: LeakyReLU slope k=%g must be finite and > 0", f, (double)ec.k);
        const int C = op == CONV_OP_FWD ? d.OC : d.IC;
        if (epi_has_stats(ec.mode)) {
            if (!ec.stats) return fail(CONV_EARG, "%s: NULL stats pointer", f);
            if ((uintptr_t)ec.stats & 7) return fail(CONV_EALIGN, "%s: stats must be 8-byte aligned", f);
            const size_t bs = (size_t)2 * C * sizeof(double);
            if (overlap(ec.stats, bs, in0, b0) || overlap(ec.stats, bs, in1, b1) || overlap(ec.stats, bs, out, bo) ||
                (ws && overlap(ec.stats, bs, ws, ws_bytes)) || (ec.A && overlap(ec.stats, bs, ec.A, bo)))
                return fail(CONV_EALIAS, "%s: stats overlaps a tensor or the workspace", f);
        }
        if (epi_reads_a(ec.mode)) {
            if (!ec.A) return fail(CONV_EARG, "%s: NULL activation pointer A", f);
            if ((uintptr_t)ec.A & 15) return fail(CONV_EALIGN, "%s: A must be 16-byte aligned", f);
            if ((ec.A != out && overlap(ec.A, bo, out, bo)) || overlap(ec.A, bo, in0, b0) || overlap(ec.A, bo, in1, b1) ||
                (ws && overlap(ec.A, bo, ws, ws_bytes)))
                return fail(CONV_EALIAS, "%s: A overlaps dY, W, the workspace, or dX other than exactly", f);
        }
    }
    if (op == CONV_OP_FWD) return run(op, in0, in1, out, d, math, ws, ws_bytes, st, ec);
    if (op == CONV_OP_BWD_DATA) return run(op, in0, in1, out, d, math, ws, ws_bytes, st, ec);
    return run(op, in1, in0, out, d, math, ws, ws_bytes, st, ec);  // dW: A = dY, B = X
}

Dims mk(int N, int IH, int IW, int IC, int OC, int FH, int FW, int sh, int sw, int ph, int pw) {
    Dims d;
    d.N = N; d.IH = IH; d.IW = IW; d.IC = IC; d.OC = OC; d.FH = FH; d.FW = FW;
    d.sh = sh; d.sw = sw; d.ph = ph; d.pw = pw; d.OH = d.OW = 0;
    return d;
}

}  // namespace

extern "C" {

int conv2d_out_hw(int IH, int IW, int FH, int FW, int sh, int sw, int ph, int pw, int* OH, int* OW) {
    if (IH < 1 || IW < 1 || FH < 1 || FW < 1 || sh < 1 || sw < 1 || ph < 0 || pw < 0 || !OH || !OW)
        return fail(CONV_EARG, "conv2d_out_hw: invalid argument");
    const long long nh = (long long)IH + 2ll * ph - FH, nw = (long long)IW + 2ll * pw - FW;
    if (nh < 0 || nw < 0) return fail(CONV_EARG, "conv2d_out_hw: kernel larger than padded input");
    *OH = (int)(nh / sh + 1);
    *OW = (int)(nw / sw + 1);
    return CONV_OK;
}

size_t conv2d_workspace_bytes(int op, int N, int IH, int IW, int IC, int OC, int FH, int FW, int sh, int sw, int ph,
                              int pw, int math) {
    Dims d = mk(N, IH, IW, IC, OC, FH, FW, sh, sw, ph, pw);
    if (check_dims(op, d, math)) return (size_t)-1;
    Plan pl;
    if (make_plan(op, d, math, pl)) return (size_t)-1;
    return pl.ws_bytes;
}

int conv2d_fwd(const float* X, const float* W, float* Y, int N, int IH, int IW, int IC, int OC, int FH, int FW,
               int sh, int sw, int ph, int pw, int math, void* ws, size_t ws_bytes, conv_stream_t st) {
    return entry(CONV_OP_FWD, X, W, Y, mk(N, IH, IW, IC, OC, FH, FW, sh, sw, ph, pw), math, ws, ws_bytes, st);
}

int conv2d_bwd_data(const float* dY, const float* W, float* dX, int N, int IH, int IW, int IC, int OC, int FH, int FW,
                    int sh, int sw, int ph, int pw, int math, void* ws, size_t ws_bytes, conv_stream_t st) {
    return entry(CONV_OP_BWD_DATA, dY, W, dX, mk(N, IH, IW, IC, OC, FH, FW, sh, sw, ph, pw), math, ws, ws_bytes, st);
}

int conv2d_bwd_filter(const float* X, const float* dY, float* dW, int N, int IH, int IW, int IC, int OC, int FH,
                      int FW, int sh, int sw, int ph, int pw, int math, void* ws, size_t ws_bytes, conv_stream_t st) {
    return entry(CONV_OP_BWD_FILTER, X, dY, dW, mk(N, IH, IW, IC, OC, FH, FW, sh, sw, ph, pw), math, ws, ws_bytes,
                 st);
}

const char* conv2d_strerror(int code) {
    switch (code) {
        case CONV_OK: return "CONV_OK";
        case CONV_EARG: return "CONV_EARG";
        case CONV_EALIGN: return "CONV_EALIGN";
        case CONV_EALIAS: return "CONV_EALIAS";
        case CONV_EWORKSPACE: return "CONV_EWORKSPACE";
        case CONV_EUNSUPPORTED: return "CONV_EUNSUPPORTED";
        case CONV_ECUDA: return "CONV_ECUDA";
        default: return "CONV_UNKNOWN";
    }
}

const char* conv2d_last_error_detail(void) { return g_detail; }

// ---------------------------------------------------------------- GEMM (include/smgemm.h)
static int gemm_check(int g, int M, int N, int K) {
    const char* f = gemm_name(g);
    if (M < 1 || N < 1 || K < 1) return fail(CONV_EARG, "%s: M=%d N=%d K=%d must be >= 1", f, M, N, K);
    const int r0 = g == 1 ? M : K;  // row lengths: matMul A[M][K], B[K][N]; T1 A[K][M]; T2 A[M][K], B[N][K]
    if (r0 % 4 || N % 4 || (g == 2 && K % 4))
        return fail(CONV_EALIGN, "%s: the row lengths (%s=%d, N=%d) must be multiples of 4 (PAPER.md:115)", f,
                    g == 1 ? "M" : "K", r0, N);
    return CONV_OK;
}

static int gemm_entry(int g, const float* A, const float* B, float* C, int M, int N, int K, int math, void* ws,
                      size_t ws_bytes, conv_stream_t st) {
    int rc = gemm_check(g, M, N, K);
    if (rc) return rc;
    g_api_name = gemm_name(g);
    {
        const GemmMap m = gemm_map(g, M, N, K);
        const int* d = m.dims;
        Dims dd = mk(d[0], d[1], d[2], d[3], d[4], d[5], d[6], d[7], d[8], d[9], d[10]);
        if (m.op == CONV_OP_FWD) rc = entry(m.op, A, B, C, dd, math, ws, ws_bytes, st);
        else if (m.op == CONV_OP_BWD_DATA) rc = entry(m.op, A, B, C, dd, math, ws, ws_bytes, st);
        else rc = entry(m.op, B, A, C, dd, math, ws, ws_bytes, st);  // dW(X = B, dY = A)
    }
    g_api_name = nullptr;
    return rc;
}

size_t gemm_workspace_bytes(int g, int M, int N, int K, int math) {
    if (g < 0 || g > 2 || gemm_check(g, M, N, K)) return (size_t)-1;
    const GemmMap m = gemm_map(g, M, N, K);
    const int* d = m.dims;
    return conv2d_workspace_bytes(m.op, d[0], d[1], d[2], d[3], d[4], d[5], d[6], d[7], d[8], d[9], d[10], math);
}

int gemm_matmul(const float* A, const float* B, float* C, int M, int N, int K, int math, void* ws, size_t ws_bytes,
                conv_stream_t st) {
    return gemm_entry(0, A, B, C, M, N, K, math, ws, ws_bytes, st);
}

int gemm_matmul_t1(const float* A, const float* B, float* C, int M, int N, int K, int math, void* ws,
                   size_t ws_bytes, conv_stream_t st) {
    return gemm_entry(1, A, B, C, M, N, K, math, ws, ws_bytes, st);
}

int gemm_matmul_t2(const float* A, const float* B, float* C, int M, int N, int K, int math, void* ws,
                   size_t ws_bytes, conv_stream_t st) {
    return gemm_entry(2, A, B, C, M, N, K, math, ws, ws_bytes, st);
}

int gemm_plan_describe(int g, int M, int N, int K, int math, char* buf, size_t len) {
    if (g < 0 || g > 2) return fail(CONV_EARG, "gemm_plan_describe: unknown gemm op %d", g);
    int rc = gemm_check(g, M, N, K);
    if (rc) return rc;
    const GemmMap m = gemm_map(g, M, N, K);
    const int* d = m.dims;
    g_api_name = gemm_name(g);
    rc = conv2d_plan_describe(m.op, d[0], d[1], d[2], d[3], d[4], d[5], d[6], d[7], d[8], d[9], d[10], math, buf,
                              len);
    g_api_name = nullptr;
    return rc;
}

// ---------------------------------------------------------------- fused epilogues (include/smconv_epi.h)
size_t conv2d_epi_workspace_bytes(int op, int N, int IH, int IW, int IC, int OC, int FH, int FW, int sh, int sw,
                                  int ph, int pw, int math, int epi) {
    Dims d = mk(N, IH, IW, IC, OC, FH, FW, sh, sw, ph, pw);
    if (check_dims(op, d, math) || epi < CONV_EPI_NONE || epi > CONV_EPI_LEAKY_BWD_STATS) return (size_t)-1;
    if (epi && !(op == CONV_OP_FWD ? (epi == CONV_EPI_BN_STATS || epi == CONV_EPI_LEAKY)
                                   : op == CONV_OP_BWD_DATA && epi_reads_a(epi)))
        return (size_t)-1;
    Plan pl;
    if (make_plan(op, d, math, pl, epi)) return (size_t)-1;
    return pl.ws_bytes;
}

int conv2d_fwd_epi(const float* X, const float* W, float* Y, double* stats, int N, int IH, int IW, int IC, int OC,
                   int FH, int FW, int sh, int sw, int ph, int pw, int math, int epi, float k, void* ws,
                   size_t ws_bytes, conv_stream_t st) {
    if (epi == CONV_EPI_LEAKY_BWD || epi == CONV_EPI_LEAKY_BWD_STATS || epi < 0 || epi > CONV_EPI_LEAKY_BWD_STATS)
        return fail(CONV_EARG, "conv2d_fwd_epi: epilogue %d is not a forward epilogue", epi);
    return entry(CONV_OP_FWD, X, W, Y, mk(N, IH, IW, IC, OC, FH, FW, sh, sw, ph, pw), math, ws, ws_bytes, st,
                 EpiCall{epi, k, nullptr, stats});
}

int conv2d_bwd_data_epi(const float* dY, const float* W, const float* A, float* dX, double* stats, int N, int IH,
                        int IW, int IC, int OC, int FH, int FW, int sh, int sw, int ph, int pw, int math, int epi,
                        float k, void* ws, size_t ws_bytes, conv_stream_t st) {
    if (epi == CONV_EPI_BN_STATS || epi == CONV_EPI_LEAKY || epi < 0 || epi > CONV_EPI_LEAKY_BWD_STATS)
        return fail(CONV_EARG, "conv2d_bwd_data_epi: epilogue %d is not a deconvolution epilogue", epi);
    return entry(CONV_OP_BWD_DATA, dY, W, dX, mk(N, IH, IW, IC, OC, FH, FW, sh, sw, ph, pw), math, ws, ws_bytes, st,
                 EpiCall{epi, k, A, stats});
}

int conv2d_epi_plan_describe(int op, int N, int IH, int IW, int IC, int OC, int FH, int FW, int sh, int sw, int ph,
                             int pw, int math, int epi, char* buf, size_t len) {
    Dims d = mk(N, IH, IW, IC, OC, FH, FW, sh, sw, ph, pw);
    int rc = check_dims(op, d, math);
    if (rc) return rc;
    if (epi < CONV_EPI_NONE || epi > CONV_EPI_LEAKY_BWD_STATS) return fail(CONV_EARG, "conv2d_epi_plan_describe: epi");
    Plan pl;
    rc = make_plan(op, d, math, pl, epi);
    if (rc) return rc;
    char base[256];
    rc = conv2d_plan_describe(op, N, IH, IW, IC, OC, FH, FW, sh, sw, ph, pw, math, base, sizeof base);
    if (rc) return rc;
    if (buf && len)
        snprintf(buf, len, "%s epi=%s groups=%d ws_epi=%zu kernels_epi=%d", base,
                 !epi ? "none" : pl.epi_fused ? "fused" : "pass", pl.epi_ngroups, pl.ws_bytes, plan_kernel_count(pl));
    return CONV_OK;
}

// ---------------------------------------------------------------- fused dW all-reduce (include/smconv_mcast.h)
size_t conv2d_bwd_filter_mcast_workspace_bytes(int N, int IH, int IW, int IC, int OC, int FH, int FW, int sh, int sw,
                                               int ph, int pw, int math) {
    Dims d = mk(N, IH, IW, IC, OC, FH, FW, sh, sw, ph, pw);
    if (check_dims(CONV_OP_BWD_FILTER, d, math)) return (size_t)-1;
    Plan pl;
    if (make_plan(CONV_OP_BWD_FILTER, d, math, pl, kMcastEpi)) return (size_t)-1;
    return pl.ws_bytes;
}

int conv2d_bwd_filter_mcast(const float* X, const float* dY, float* dW_mc, int N, int IH, int IW, int IC, int OC, int FH,
                            int FW, int sh, int sw, int ph, int pw, int math, void* ws, size_t ws_bytes,
                            conv_stream_t st) {
    g_api_name = "conv2d_bwd_filter_mcast";
    const int rc = entry(CONV_OP_BWD_FILTER, X, dY, dW_mc, mk(N, IH, IW, IC, OC, FH, FW, sh, sw, ph, pw), math, ws,
                         ws_bytes, st, kMcastCall);
    g_api_name = nullptr;
    return rc;
}

int conv2d_bwd_filter_mcast_plan_describe(int N, int IH, int IW, int IC, int OC, int FH, int FW, int sh, int sw,
                                          int ph, int pw, int math, char* buf, size_t len) {
    Dims d = mk(N, IH, IW, IC, OC, FH, FW, sh, sw, ph, pw);
    int rc = check_dims(CONV_OP_BWD_FILTER, d, math);
    if (rc) return rc;
    Plan pl;
    rc = make_plan(CONV_OP_BWD_FILTER, d, math, pl, kMcastEpi);
    if (rc) return rc;
    if (buf && len)
        snprintf(buf, len, "variant=%d BN=%d splits=%d mcast=%s ws=%zu kernels=%d", pl.variant, pl.BN, pl.splits,
                 pl.mc_direct ? "epilogue" : "reduce", pl.ws_bytes, plan_kernel_count(pl));
    return CONV_OK;
}

int smconv_set_pair(int on) { return tma_set_pair(on ? 1 : 0); }

int smconv_set_trace(void* device_buf) {
    g_trace.store((unsigned long long*)device_buf);
    return CONV_OK;
}

double smconv_set_hybrid_min_gflop(double gflop) {
    const double old = g_hyb_min_gflop.exchange(gflop);
    std::lock_guard<std::mutex> lk(g_plan_mu);
    g_plans.clear();  // plans depend on it
    return old;
}

int conv2d_force_variant(int op, int variant) {
    if (op < 0 || op > 2 || variant < 0 || variant > 6) return fail(CONV_EARG, "conv2d_force_variant: bad op/variant");
    read_env_once();
    g_force[op].store(variant);
    return CONV_OK;
}

int conv2d_plan_describe(int op, int N, int IH, int IW, int IC, int OC, int FH, int FW, int sh, int sw, int ph,
                         int pw, int math, char* buf, size_t len) {
    Dims d = mk(N, IH, IW, IC, OC, FH, FW, sh, sw, ph, pw);
    int rc = check_dims(op, d, math);
    if (rc) return rc;
    Plan pl;
    rc = make_plan(op, d, math, pl);
    if (rc) return rc;
    if (buf && len)
        snprintf(buf, len, "variant=%s%s%s%s%s BN=%d planes=%d splits=%d grid=%ux%ux%u ws=%zu kernels=%d",
                 pl.s2dx ? "tma s2dx" :
                 pl.variant == CONV_VARIANT_DWS      ? "dws"
                 : pl.variant == CONV_VARIANT_STEM   ? "stem"
                 : pl.variant == CONV_VARIANT_DIRECT ? "direct"
                 : pl.variant == CONV_VARIANT_STRIP ? "strip"
                 : pl.variant == CONV_VARIANT_TMA   ? "tma"
                                                    : "generic",
                 ((pl.variant == CONV_VARIANT_TMA && pl.tp.pair) ||
                  (pl.variant == CONV_VARIANT_STRIP && strip_pair(op, N, pl.BN, pl.planes)) ||
                  (pl.variant == CONV_VARIANT_DWS && dws_pair_mode()))
                     ? " pair=2cta"
                     : "", pl.gp.csk ? " csk" : "",
                 (pl.variant == CONV_VARIANT_TMA && pl.planes == 2 && op != CONV_OP_BWD_FILTER && !pl.gp.hyb) ? " 3mma"
                                                                                                              : "",
                 (pl.variant == CONV_VARIANT_TMA && pl.tp.zf1) ? " zfill"
                 : ((pl.variant == CONV_VARIANT_TMA && pl.tp.dw_hyb) ||
                    (pl.variant == CONV_VARIANT_DWS && pl.planes == 2 && dws_hyb_mode())) ? " hybw" : "",
                 pl.BN, pl.planes, pl.splits, pl.grid.x,
                 pl.grid.y, pl.grid.z, pl.ws_bytes, plan_kernel_count(pl));
    return CONV_OK;
}

int conv2d_plan_kernels(int op, int N, int IH, int IW, int IC, int OC, int FH, int FW, int sh, int sw, int ph, int pw,
                        int math) {
    Dims d = mk(N, IH, IW, IC, OC, FH, FW, sh, sw, ph, pw);
    if (check_dims(op, d, math)) return -1;
    Plan pl;
    if (make_plan(op, d, math, pl)) return -1;
    return plan_kernel_count(pl);
}

int smconv_selftest_host(void) {
    // fast division must equal integer division for every divisor / dividend we use
    const uint32_t ds[] = {1, 2, 3, 4, 5, 6, 7, 8, 9, 11, 12, 16, 17, 25, 31, 32, 33, 64, 100, 121, 128, 192, 255,
                           256, 257, 480, 512, 528, 832, 1000, 1024, 4096, 65535, 65536, 1000003};
    for (uint32_t d : ds) {
        FastDiv f = make_fastdiv(d);
        uint32_t n = 0;
        for (int i = 0; i < 200000; ++i) {
            if (fdiv(n, f) != n / d) return 1;
            n = (n * 1103515245u + 12345u) & 0x7FFFFFFFu;
        }
        for (uint32_t k = 0; k < 4096; ++k) {
            const uint32_t m = k * d;
            if (m >= 0x80000000u) break;
            if (fdiv(m, f) != k || (m && fdiv(m - 1, f) != k - 1)) return 2;
        }
        if (fdiv(0x7FFFFFFFu, f) != 0x7FFFFFFFu / d) return 3;
    }
    return 0;
}

}  // extern "C"
