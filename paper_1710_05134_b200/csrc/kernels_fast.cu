// kernels_fast.cu — row a4 of SURVEY.md §8: the Schur-complement update of the
// contribution block, CB -= L_CB W_CB^T over all eliminated pivots of a front
// (BASELINE north_star part (4): "the one genuine dense contraction").
//
// k_schur: one CTA per 64x64 lower tile of each CB of a level, K = #eliminated;
// operands staged through shared memory with cp.async (double buffered),
// FP64 tensor-core inner product (mma.sync m8n8k4 f64 = SASS DMMA).
// Storage: L[i,t] at F[i + t*ld] (lower), W[i,t] at F[t + i*ld] (upper).
#include <cfloat>
#include <cstdlib>
#include <climits>
#include <cstdint>

#include <cudaTypedefs.h>

#include "device.cuh"

namespace kep {

namespace {

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

constexpr int ST = 64;          // CTA tile (rows and cols)
constexpr int KC = 16;          // K chunk per pipeline stage
constexpr int APAD = 68;        // A smem row stride (doubles): = 4 (mod 16), conflict-free f64 fragments
constexpr int BPAD = 20;        // B smem row stride (doubles)
constexpr int SCH_T = 128;      // 4 warps, 2 x 2 of 32 x 32

__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
    const int sz = valid ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(src), "r"(sz));
}
// 16-byte copy (two doubles), `bytes` in {0, 8, 16} valid source bytes, the rest zero-filled
__device__ __forceinline__ void cp_async16(double* dst, const double* src, int bytes) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(src), "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__global__ void __launch_bounds__(SCH_T) k_schur(DevPlan P, const int4* __restrict__ items) {
    // CB -= L21 D L21^T = G S G^T: both operands are rows of G (upper part, written by
    // k_l21), S = diag(+-1) applied to the B fragments as sign-bit flips (no FP64 work).
    __shared__ __align__(16) double As[2][ST][BPAD];      // [row][t]: G rows of the tile's CB rows
    __shared__ __align__(16) double Bs[2][ST][BPAD];      // [col][t]: G rows of the tile's CB columns
    __shared__ unsigned long long Sg[2][KC];
    const int4 it = items[blockIdx.x];          // (front, I, J, -)
    const int s = it.x, I = it.y, J = it.z;
    const int sh = blockIdx.y;
    const int nd = P.nd_in[(size_t)sh * P.nf + s];
    if (nd < 0) return;
    if (P.flag[(size_t)sh * P.nf + s] != FL_OK) return;   // redone by the unblocked kernel (CB updated there)
    const int ndo = P.nd_out[(size_t)sh * P.nf + s];
    const int p = P.npiv[s], c = P.ncb[s];
    const int f = P.forder[s] + nd, q = p + nd, ld = ldpad(P.cap[s]);
    const int e = q - ndo;                       // eliminated pivots = K
    if (e <= 0) return;
    double* F = P.arena + (size_t)sh * P.arena_stride + P.arena_off[s];
    const AuxRec A = aux_rec(P, sh, s, P.cap[s] - c);
    const int r0 = q + I * ST, c0 = q + J * ST;  // tile origin (front positions)
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, tg = lane & 3;
    const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
    auto load = [&](int buf, int t0) {
        // rows are 16-byte aligned (even leading dimension): one 16-byte copy per pair of pivots
        for (int x = tid; x < ST * (KC / 2); x += SCH_T) {
            const int i = x / (KC / 2), tt = 2 * (x - i * (KC / 2));
            const int gt = t0 + tt;
            const int gi = r0 + i, gj = c0 + i;
            const int nv = gt + 1 < e ? 16 : (gt < e ? 8 : 0);
            const int na = gi < f ? nv : 0, nb = gj < f ? nv : 0;
            cp_async16(&As[buf][i][tt], F + (na ? (gt + (size_t)gi * ld) : 0), na);
            cp_async16(&Bs[buf][i][tt], F + (nb ? (gt + (size_t)gj * ld) : 0), nb);
        }
        if (tid < KC) Sg[buf][tid] = (t0 + tid < e && A.sgn[t0 + tid] < 0.0) ? 0x8000000000000000ull : 0ull;
        cp_async_commit();
    };
    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    const int nk = (e + KC - 1) / KC;
    load(0, 0);
    for (int kc = 0; kc < nk; ++kc) {
        const int buf = kc & 1;
        if (kc + 1 < nk) {
            load(buf ^ 1, (kc + 1) * KC);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
#pragma unroll
        for (int k4 = 0; k4 < KC; k4 += 4) {
            double a[4], b[4];
#pragma unroll
            for (int mb = 0; mb < 4; ++mb) a[mb] = As[buf][wm + 8 * mb + g][k4 + tg];
#pragma unroll
            for (int nb = 0; nb < 4; ++nb)
                b[nb] = __longlong_as_double(__double_as_longlong(Bs[buf][wn + 8 * nb + g][k4 + tg]) ^ (long long)Sg[buf][k4 + tg]);
#pragma unroll
            for (int mb = 0; mb < 4; ++mb)
#pragma unroll
                for (int nb = 0; nb < 4; ++nb) dmma(acc[mb][nb], a[mb], b[nb]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int mb = 0; mb < 4; ++mb)
#pragma unroll
        for (int nb = 0; nb < 4; ++nb)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int i = r0 + wm + 8 * mb + g;
                const int j = c0 + wn + 8 * nb + 2 * tg + h;
                if (i < f && j < f && i >= j) atomicAdd(&F[i + (size_t)j * ld], -acc[mb][nb][h]);   // one writer: RED, no load wait
            }
}

// ---------------------------------------------------------------- k_schur_tma
// The same tile computation fed by TMA (cp.async.bulk.tensor, SASS UTMALDG): per K
// chunk of 16 pivots, one elected thread issues two 16 x 64 boxes (the G rows of the
// tile's CB rows and of its CB columns) from the front's tensor map into a 128-byte
// swizzled stage and arms the stage's "full" mbarrier with the byte count; the four
// warps wait on it, run the DMMA k-steps and arrive on the stage's "empty" mbarrier;
// the producer refills a stage once it is empty.  KST stages in flight, no CTA-wide
// barrier in the K loop.  Columns t >= e of the last chunk (other data of the front)
// are masked on the B fragments together with the D-sign flip.
constexpr int KST = 3;                        // pipeline stages (48 KB: 4 CTAs per SM)
constexpr int TBOX = ST * KC;                 // doubles per box (64 rows x 16 pivots, 8 KB)

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
        ::"r"(smem_u32(dst)), "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar)) : "memory");
}
// element (row, t) of a 64 x 16 box stored with the 128-byte swizzle: 16-byte chunk (t / 2) ^ (row % 8)
__device__ __forceinline__ int swz(int row, int t) { return row * KC + ((((t >> 1) ^ (row & 7)) << 1) | (t & 1)); }

__global__ void __launch_bounds__(SCH_T, 4) k_schur_tma(DevPlan P, const int4* __restrict__ items) {
    extern __shared__ __align__(1024) unsigned char tsm[];
    const unsigned pad = (1024u - (smem_u32(tsm) & 1023u)) & 1023u;  // the 128-byte swizzle atom is 1 KB
    double* As = reinterpret_cast<double*>(tsm + pad);            // [KST][64][16] swizzled
    double* Bs = As + KST * TBOX;                                 // [KST][64][16]
    __shared__ __align__(8) uint64_t full[KST], empty[KST];
    const int4 it = items[blockIdx.x];
    const int s = it.x, I = it.y, J = it.z;
    const int sh = blockIdx.y;
    const int nd = P.nd_in[(size_t)sh * P.nf + s];
    if (nd < 0) return;
    if (P.flag[(size_t)sh * P.nf + s] != FL_OK) return;
    const int ndo = P.nd_out[(size_t)sh * P.nf + s];
    const int p = P.npiv[s], c = P.ncb[s];
    const int f = P.forder[s] + nd, q = p + nd, ld = ldpad(P.cap[s]);
    const int e = q - ndo;
    if (e <= 0) return;
    const int r0 = q + I * ST, c0 = q + J * ST;
    if (r0 >= f) return;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, tg = lane & 3;
    const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
    const CUtensorMap* map = P.tmaps + (size_t)sh * P.ntmap + P.tmap_idx[s];
    const int ybase = (int)(P.arena_off[s] / ld);                 // the front starts at a multiple of ld
    const AuxRec A = aux_rec(P, sh, s, P.cap[s] - c);
    const int nk = (e + KC - 1) / KC;
    if (tid == 0) {
        for (int k = 0; k < KST; ++k) { mbar_init(&full[k], 1); mbar_init(&empty[k], SCH_T / 32); }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(map) : "memory");
    }
    __syncthreads();
    auto issue = [&](int kc) {
        const int st = kc % KST;
        mbar_expect_tx(&full[st], 2 * TBOX * sizeof(double));
        tma_load_2d(As + st * TBOX, map, kc * KC, ybase + r0, &full[st]);
        tma_load_2d(Bs + st * TBOX, map, kc * KC, ybase + c0, &full[st]);
    };
    if (tid == 0)
        for (int kc = 0; kc < KST && kc < nk; ++kc) issue(kc);
    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    for (int kc = 0; kc < nk; ++kc) {
        const int st = kc % KST;
        // masks of this chunk's pivots (t = kc KC + 4 k4 + tg): bit k4 keep (t < e), bit 4 + k4 sign of D
        unsigned msk = 0;
#pragma unroll
        for (int k4 = 0; k4 < 4; ++k4) {
            const int t = kc * KC + 4 * k4 + tg;
            if (t < e) msk |= (1u << k4) | (A.sgn[t] < 0.0 ? (16u << k4) : 0u);
        }
        mbar_wait(&full[st], (unsigned)((kc / KST) & 1));
        const double* as = As + st * TBOX;
        const double* bs = Bs + st * TBOX;
#pragma unroll
        for (int k4 = 0; k4 < 4; ++k4) {
            double a[4], b[4];
            const long long keep = ((msk >> k4) & 1u) ? -1ll : 0ll;
            const long long sgn = (long long)((unsigned long long)((msk >> (4 + k4)) & 1u) << 63);
#pragma unroll
            for (int mb = 0; mb < 4; ++mb) a[mb] = as[swz(wm + 8 * mb + g, 4 * k4 + tg)];
#pragma unroll
            for (int nb = 0; nb < 4; ++nb)
                b[nb] = __longlong_as_double((__double_as_longlong(bs[swz(wn + 8 * nb + g, 4 * k4 + tg)]) & keep) ^ sgn);
#pragma unroll
            for (int mb = 0; mb < 4; ++mb)
#pragma unroll
                for (int nb = 0; nb < 4; ++nb) dmma(acc[mb][nb], a[mb], b[nb]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
        if (tid == 0 && kc + KST < nk) {                        // refill this stage once every warp is done
            mbar_wait(&empty[st], (unsigned)((kc / KST) & 1));
            issue(kc + KST);
        }
    }
#pragma unroll
    for (int mb = 0; mb < 4; ++mb)
#pragma unroll
        for (int nb = 0; nb < 4; ++nb)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int i = r0 + wm + 8 * mb + g;
                const int j = c0 + wn + 8 * nb + 2 * tg + h;
                double* F = P.arena + (size_t)sh * P.arena_stride + P.arena_off[s];
                if (i < f && j < f && i >= j) atomicAdd(&F[i + (size_t)j * ld], -acc[mb][nb][h]);
            }
}

// Small fronts (c <= 256, FS block <= 48): one CTA per front, the CB's G rows
// staged in shared memory once, every 32 x 32 lower tile of the CB computed from
// them (DMMA), RED epilogue.  Avoids the per-tile setup and the repeated operand
// loads of k_schur where K (= pivots) is a single chunk.
constexpr int SS_T = 256;
constexpr int SS_C = 256;       // max CB order
constexpr int SS_K = 48;        // max eliminated pivots
constexpr int SS_P = SS_K + 4;  // = 4 (mod 16)
constexpr int SS_QMAX = 128;   // eliminated pivots at most (k_small's FS limit)

template <bool RED>
__global__ void __launch_bounds__(SS_T) k_schur_small(DevPlan P, const int32_t* __restrict__ fronts, int SP) {
    extern __shared__ __align__(16) double Gs[];        // [c][SP], SP = 4 (mod 16) >= K4 of the level's fronts
    __shared__ unsigned long long Sg[SS_QMAX];
    const int s = fronts[blockIdx.x];
    const int sh = blockIdx.y;
    const int nd = P.nd_in[(size_t)sh * P.nf + s];
    if (nd < 0) return;
    if (P.flag[(size_t)sh * P.nf + s] != FL_OK) return;
    const int ndo = P.nd_out[(size_t)sh * P.nf + s];
    const int p = P.npiv[s], c = P.ncb[s];
    const int f = P.forder[s] + nd, q = p + nd, ld = ldpad(P.cap[s]);
    const int e = q - ndo;
    if (e <= 0 || c <= 0 || e > SS_QMAX) return;       // (e <= 128: k_small's limit; FS capacity <= SS_K otherwise)
    double* F = P.arena + (size_t)sh * P.arena_stride + P.arena_off[s];
    const AuxRec A = aux_rec(P, sh, s, P.cap[s] - c);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, tg = lane & 3;
    const int K4 = (e + 3) & ~3;
    // K chunk held in shared memory: one chunk unless a k_small front received more delayed columns
    // than its plan (its pivot count can then exceed the level's planned maximum)
    const int KW = SP - 4;
    for (int t = tid; t < SS_QMAX; t += SS_T) Sg[t] = (t < e && A.sgn[t] < 0.0) ? 0x8000000000000000ull : 0ull;
    const int T = (c + 31) >> 5;
    const int ntile = T * (T + 1) / 2;
    for (int kc0 = 0; kc0 < K4; kc0 += KW) {
        const int kw = min(KW, K4 - kc0);
        __syncthreads();                                 // previous chunk consumed (and Sg written)
        for (int x = tid; x < c * kw; x += SS_T) {       // G rows of the CB (upper part), zero-padded to K4
            const int i = x / kw, t = x - i * kw;
            const bool v = kc0 + t < e;
            cp_async8(&Gs[i * SP + t], F + (v ? (kc0 + t + (size_t)(q + i) * ld) : 0), v);
        }
        cp_async_commit();
        cp_async_wait<0>();
        __syncthreads();
        for (int tile = warp; tile < ntile; tile += SS_T / 32) {
            int I = (int)((sqrtf(8.0f * tile + 1.0f) - 1.0f) * 0.5f);
            while ((I + 1) * (I + 2) / 2 <= tile) ++I;
            while (I * (I + 1) / 2 > tile) --I;
            const int J = tile - I * (I + 1) / 2;
            const int i0 = 32 * I, j0 = 32 * J;
            double acc[4][4][2];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
            for (int k4 = 0; k4 < kw; k4 += 4) {
                double a[4], b[4];
                const long long sm = (long long)Sg[kc0 + k4 + tg];
#pragma unroll
                for (int mb = 0; mb < 4; ++mb) {
                    const int i = i0 + 8 * mb + g;
                    a[mb] = i < c ? Gs[i * SP + k4 + tg] : 0.0;
                }
#pragma unroll
                for (int nb = 0; nb < 4; ++nb) {
                    const int j = j0 + 8 * nb + g;
                    b[nb] = j < c ? __longlong_as_double(__double_as_longlong(Gs[j * SP + k4 + tg]) ^ sm) : 0.0;
                }
#pragma unroll
                for (int mb = 0; mb < 4; ++mb)
#pragma unroll
                    for (int nb = 0; nb < 4; ++nb) dmma(acc[mb][nb], a[mb], b[nb]);
            }
#pragma unroll
            for (int mb = 0; mb < 4; ++mb)
#pragma unroll
                for (int nb = 0; nb < 4; ++nb)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int i = i0 + 8 * mb + g;
                        const int j = j0 + 8 * nb + 2 * tg + h;
                        if (i < c && j < c && i >= j) {
                            double* x = &F[(q + i) + (size_t)(q + j) * ld];
                            if (RED) atomicAdd(x, -acc[mb][nb][h]);
                            else *x -= acc[mb][nb][h];                     // the tile's only writer
                        }
                    }
        }
    }
}

}  // namespace

void launch_schur(const DevPlan& P, const int4* items, int nitems, int batch, cudaStream_t st) {
    if (nitems <= 0) return;
    k_schur<<<dim3(nitems, batch), SCH_T, 0, st>>>(P, items);
}

void launch_schur_tma(const DevPlan& P, const int4* items, int nitems, int batch, cudaStream_t st) {
    if (nitems <= 0) return;
    const size_t smem = 2 * KST * TBOX * sizeof(double) + 1024;     // + alignment slack for the 1 KB swizzle atom
    static unsigned long long attr = 0;
    if (first_on_device(attr)) cudaFuncSetAttribute(k_schur_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_schur_tma<<<dim3(nitems, batch), SCH_T, smem, st>>>(P, items);
}

}  // namespace kep

namespace kep {
bool encode_front_tmap(CUtensorMap* out, double* base, int64_t arena_doubles, int ld) {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !ptr) {
            cudaGetLastError();
            return false;
        }
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    }
    const cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)(arena_doubles / ld)};
    const cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(double)};
    const cuuint32_t box[2] = {(cuuint32_t)KC, (cuuint32_t)ST};
    const cuuint32_t es[2] = {1, 1};
    const CUresult r = fn(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, base, dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

bool schur_small_ok(int c, int qcap) { return c > 0 && c <= SS_C && qcap <= SS_K; }

void launch_schur_small(const DevPlan& P, const int32_t* fronts, int nfronts, int batch, int cmax, int kmax,
                        cudaStream_t st) {
    if (nfronts <= 0) return;
    // shared memory sized for the level's largest CB and planned pivot count, not the kernel maxima
    const int SP = ((((kmax + 3) & ~3) + 15) & ~15) + 4;       // >= K4, = 4 (mod 16)
    const size_t smem = sizeof(double) * (size_t)std::min(cmax, SS_C) * SP;
    const size_t smax = sizeof(double) * SS_C * SS_P;           // the opt-in covers every level
    static unsigned long long attr = 0;
    if (first_on_device(attr)) {
        cudaFuncSetAttribute(k_schur_small<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smax);
        cudaFuncSetAttribute(k_schur_small<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smax);
    }
    static const bool red = getenv("KEP_SCHUR_NORED") == nullptr;   // RED measured 2.6x faster at c4 level 0
    if (red) k_schur_small<true><<<dim3(nfronts, batch), SS_T, smem, st>>>(P, fronts, SP);
    else k_schur_small<false><<<dim3(nfronts, batch), SS_T, smem, st>>>(P, fronts, SP);
}
}  // namespace kep
