/*
 * CPU ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the two numba kernels of the reference package,
 * compiled with -ffp-contract=off so every multiply and add rounds
 * separately, exactly as the numba (LLVM, no fastmath) originals do.
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may
 * load this library; the product path never does.
 *
 *   oracle_matmul      restates numkit._mm_kernel   (numkit.py:78-90)
 *   oracle_fk_compose  restates bodymodel._fk_compose (bodymodel.py:208-240)
 */
#include <stdint.h>

/* C[m,n] = A[m,k] @ B[k,n]; every C[i,j] is the left-to-right sum over k
 * starting from +0, one rounding per product and per add. */
void oracle_matmul(const float *a, const float *b, float *c,
                   int64_t m, int64_t k, int64_t n)
{
    for (int64_t i = 0; i < m; ++i) {
        float *row = c + i * n;
        for (int64_t j = 0; j < n; ++j)
            row[j] = 0.0f;
        for (int64_t p = 0; p < k; ++p) {
            const float s = a[i * k + p];
            const float *brow = b + p * n;
            for (int64_t j = 0; j < n; ++j)
                row[j] += s * brow[j];
        }
    }
}

/* Kinematic chain for one pose: world rotations/translations in joint order
 * and the rest-relative translation t_w - R_w g_rest. */
void oracle_fk_compose(const float *rot_local /* nj*9 */,
                       const float *t_local /* nj*3 */,
                       const int64_t *parents, const float *rest /* nj*3 */,
                       float *rot_w /* nj*9 */, float *t_w /* nj*3 */,
                       float *at /* nj*3 */, int64_t nj)
{
    for (int64_t j = 0; j < nj; ++j) {
        const int64_t p = parents[j];
        const float *rl = rot_local + 9 * j;
        float *rj = rot_w + 9 * j;
        if (p < 0) {
            for (int e = 0; e < 9; ++e) rj[e] = rl[e];
            for (int a = 0; a < 3; ++a) t_w[3 * j + a] = t_local[3 * j + a];
        } else {
            const float *rp = rot_w + 9 * p;
            for (int a = 0; a < 3; ++a) {
                for (int b = 0; b < 3; ++b) {
                    float s = rp[3 * a + 0] * rl[0 * 3 + b];
                    s += rp[3 * a + 1] * rl[1 * 3 + b];
                    s += rp[3 * a + 2] * rl[2 * 3 + b];
                    rj[3 * a + b] = s;
                }
                float s = rp[3 * a + 0] * t_local[3 * j + 0];
                s += rp[3 * a + 1] * t_local[3 * j + 1];
                s += rp[3 * a + 2] * t_local[3 * j + 2];
                t_w[3 * j + a] = s + t_w[3 * p + a];
            }
        }
        for (int a = 0; a < 3; ++a) {
            float s = rj[3 * a + 0] * rest[3 * j + 0];
            s += rj[3 * a + 1] * rest[3 * j + 1];
            s += rj[3 * a + 2] * rest[3 * j + 2];
            at[3 * j + a] = t_w[3 * j + a] - s;
        }
    }
}
