/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the einsum / linalg.generic
 * hot path.  Nothing in the product path (paper_2503_04771_b200/) links or
 * calls this file; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs do, and only as the checker.
 *
 * It restates, in plain C, the reference evaluator's loop nest
 *   /root/reference/pkg/src/bridgegen/interp.py:372-424  (_Machine._generic)
 * with the per-point body synthesised by
 *   /root/reference/pkg/src/bridgegen/einsum.py:100-118  (_body_function)
 * and the scalar IEEE semantics of
 *   /root/reference/pkg/src/bridgegen/interp.py:260-274  (arith.mulf / addf)
 *
 * Semantics reproduced exactly (and pinned bit-for-bit against the reference
 * by tests/test_oracle.py on the tests/golden fixtures):
 *   - axes = output indices, then input-only indices (einsum.py:81), so every
 *     output element owns one contiguous lexicographic run of the reduction
 *     sub-space (interp.py:407-420 recurses in axis order);
 *   - result starts as a copy of the output operand (interp.py:399);
 *   - per point: p = x1; p = fl(p * xk) for k = 2..n (left fold,
 *     einsum.py:111-116); acc = fl(p + acc) (einsum.py:116-117);
 *   - one input with no reduction axis is a passthrough: out = x1
 *     (einsum.py:105-108) — the initial output value is ignored.
 * Every multiply and add is a separately rounded binary32/binary64 op:
 * compiled with -ffp-contract=off and without fast-math (no FMA contraction,
 * no reassociation, no flush-to-zero).  Parallelism (OpenMP) is over output
 * elements only, which keeps each element's reduction order — and therefore
 * its bits — identical to the reference's sequential loop.
 *
 * The one reference behaviour NOT reproduced: the reference round-trips
 * scalars through Python float, which quiets signalling NaNs.
 * This oracle, like the GPU kernels, moves bits unchanged.
 */
#include <stdint.h>
#include <string.h>
#include <omp.h>   /* built with -fopenmp (oracle/Makefile) */

#define ORACLE_MAX_AXES 16
#define ORACLE_MAX_OPERANDS 8

/*
 * Generic loop nest.
 *   n_in        number of input operands (1..8)
 *   n_axes      number of iteration axes (parallel first, then reduction)
 *   n_par       number of parallel (= output) axes
 *   extents     [n_axes]
 *   ins         [n_in] base pointers
 *   strides     [n_in * n_axes] element stride of operand k along axis a
 *               (0 when the operand does not index that axis)
 *   c0          initial output, row-major over the parallel axes
 *   out         result, row-major over the parallel axes (may alias c0)
 *   o_begin/o_end  half-open range of output linear indices to compute
 *               (lets callers time a bounded sample of a huge job)
 *   threads     OpenMP threads (<=0: library default)
 */
#define DEFINE_GENERIC(NAME, T)                                                \
int NAME(int n_in, int n_axes, int n_par, const int64_t *extents,              \
         const T *const *ins, const int64_t *strides, const T *c0, T *out,     \
         int64_t o_begin, int64_t o_end, int threads)                          \
{                                                                              \
    if (n_in < 1 || n_in > ORACLE_MAX_OPERANDS) return -1;                     \
    if (n_axes < 0 || n_axes > ORACLE_MAX_AXES || n_par > n_axes) return -1;   \
    const int n_red = n_axes - n_par;                                          \
    const int passthrough = (n_in == 1 && n_red == 0);                         \
    int64_t red_points = 1;                                                    \
    for (int a = n_par; a < n_axes; ++a) red_points *= extents[a];             \
    (void)threads;                                                             \
    _Pragma("omp parallel for schedule(dynamic, 16) num_threads(threads > 0 ? threads : omp_get_max_threads())") \
    for (int64_t o = o_begin; o < o_end; ++o) {                                \
        /* decode the parallel coordinates of output element o */             \
        int64_t base[ORACLE_MAX_OPERANDS];                                     \
        for (int k = 0; k < n_in; ++k) base[k] = 0;                            \
        int64_t rem = o;                                                       \
        for (int a = n_par - 1; a >= 0; --a) {                                 \
            int64_t i = rem % extents[a];                                      \
            rem /= extents[a];                                                 \
            for (int k = 0; k < n_in; ++k) base[k] += i * strides[k * n_axes + a]; \
        }                                                                      \
        if (passthrough) { out[o] = ins[0][base[0]]; continue; }               \
        T acc = c0[o];                                                         \
        if (red_points == 0) { out[o] = acc; continue; }                       \
        int64_t idx[ORACLE_MAX_AXES];                                          \
        int64_t off[ORACLE_MAX_OPERANDS];                                      \
        for (int a = 0; a < n_red; ++a) idx[a] = 0;                            \
        for (int k = 0; k < n_in; ++k) off[k] = base[k];                       \
        for (int64_t r = 0; r < red_points; ++r) {                             \
            T p = ins[0][off[0]];                                              \
            for (int k = 1; k < n_in; ++k) p = p * ins[k][off[k]];                 \
            acc = p + acc;                                                     \
            /* odometer over the reduction axes, last axis fastest */          \
            for (int a = n_red - 1; a >= 0; --a) {                             \
                const int ax = n_par + a;                                      \
                if (++idx[a] < extents[ax]) {                                  \
                    for (int k = 0; k < n_in; ++k) off[k] += strides[k * n_axes + ax]; \
                    break;                                                     \
                }                                                              \
                for (int k = 0; k < n_in; ++k)                                 \
                    off[k] -= (extents[ax] - 1) * strides[k * n_axes + ax];    \
                idx[a] = 0;                                                    \
            }                                                                  \
        }                                                                      \
        out[o] = acc;                                                          \
    }                                                                          \
    return 0;                                                                  \
}

DEFINE_GENERIC(oracle_generic_f32, float)
DEFINE_GENERIC(oracle_generic_f64, double)

/*
 * Two-operand contraction with a single (flattened) reduction group, batched:
 *   out[b,m,n] = fl(... fl(fl(A[b,m,0]*B[b,0,n]) + C0[b,m,n]) ...)  k = 0..K-1
 * i.e. exactly the generic loop above for specs like (b,i,k),(b,k,j)->(b,i,j),
 * but with the loops ordered (m, k, n) so the n loop vectorises.  Each output
 * element still sees its products in increasing k with separate rounding, so
 * the bits equal the reference's (tests/test_oracle.py pins this).
 * Strides are in elements: A (sab, sam, sak), B (sbb, sbk, sbn); C0/out are
 * dense row-major [batch, M, N].  Rows [m_begin, m_end) of every batch.
 */
int oracle_gemm_kseq_f32(int64_t batch, int64_t M, int64_t N, int64_t K,
                         const float *A, int64_t sab, int64_t sam, int64_t sak,
                         const float *B, int64_t sbb, int64_t sbk, int64_t sbn,
                         const float *c0, float *out,
                         int64_t m_begin, int64_t m_end, int threads)
{
    if (m_end > M) m_end = M;
    if (m_begin < 0) m_begin = 0;
    const int64_t rows = m_end - m_begin;
    if (rows <= 0) return 0;
    (void)threads;
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads > 0 ? threads : omp_get_max_threads())
    for (int64_t t = 0; t < batch * rows; ++t) {
        const int64_t b = t / rows, m = m_begin + t % rows;
        float *o = out + (b * M + m) * N;
        const float *c = c0 + (b * M + m) * N;
        if (o != c) memcpy(o, c, sizeof(float) * (size_t)N);
        const float *a = A + b * sab + m * sam;
        const float *bb = B + b * sbb;
        for (int64_t k = 0; k < K; ++k) {
            const float av = a[k * sak];
            const float *brow = bb + k * sbk;
            if (sbn == 1) {
                for (int64_t n = 0; n < N; ++n) { float p = av * brow[n]; o[n] = p + o[n]; }
            } else {
                for (int64_t n = 0; n < N; ++n) { float p = av * brow[n * sbn]; o[n] = p + o[n]; }
            }
        }
    }
    return 0;
}

int oracle_version(void) { return 1; }

/*
 * The BASELINE config-5 chain (i,k),(k,j),(j,l)->(i,l) with the reference's
 * UNFACTORED per-point semantics: axes (i, l, k, j) (einsum.py:81), so each
 * output element accumulates, for k outer and j inner,
 *     p = fl(a[i,k] * b[k,j]); p = fl(p * c[j,l]); acc = fl(p + acc)
 * exactly as oracle_generic_f32 / the reference do — but 16 consecutive l are
 * carried in 16 independent accumulators so the inner loop vectorises over l
 * (c rows are contiguous).  Each lane's operation sequence is unchanged, so
 * the bits equal oracle_generic_f32's (tests/test_oracle.py).  Row-major
 * dense a (I x K), b (K x J), c (J x L), out (I x L) initialised by caller.
 * Computes rows [i0, i1) x columns [l0, l1).
 */
#define CHAIN_LANES 16
int oracle_chain3_f32(int64_t I, int64_t K, int64_t J, int64_t L,
                      const float *a, const float *b, const float *c, float *out,
                      int64_t i0, int64_t i1, int64_t l0, int64_t l1, int threads)
{
    (void)I;
    const int64_t nlb = (l1 - l0 + CHAIN_LANES - 1) / CHAIN_LANES;
    const int64_t tasks = (i1 - i0) * nlb;
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads > 0 ? threads : omp_get_max_threads())
    for (int64_t t = 0; t < tasks; ++t) {
        const int64_t i = i0 + t / nlb;
        const int64_t lb = l0 + (t % nlb) * CHAIN_LANES;
        const int64_t nl = (l1 - lb) < CHAIN_LANES ? (l1 - lb) : CHAIN_LANES;
        float acc[CHAIN_LANES];
        for (int q = 0; q < CHAIN_LANES; ++q) acc[q] = q < nl ? out[i * L + lb + q] : 0.0f;
        for (int64_t k = 0; k < K; ++k) {
            const float aik = a[i * K + k];
            const float *brow = b + k * J;
            for (int64_t j = 0; j < J; ++j) {
                const float p = aik * brow[j];
                const float *crow = c + j * L + lb;
                if (nl == CHAIN_LANES) {
                    for (int q = 0; q < CHAIN_LANES; ++q) acc[q] = p * crow[q] + acc[q];
                } else {
                    for (int q = 0; q < nl; ++q) acc[q] = p * crow[q] + acc[q];
                }
            }
        }
        for (int q = 0; q < nl; ++q) out[i * L + lb + q] = acc[q];
    }
    return 0;
}
