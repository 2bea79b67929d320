/*
 * spx_oracle.c -- CPU ORACLE for the libspx GPU kernels.  TEST
 * INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
 * cpu_baseline / `--impl reference` legs of bench.py, never by the product.
 *
 * A plain-C restatement of the reference semantics of the hot path:
 *   - SearchSegment / SearchCoord           ir.py:178-205
 *   - the multi-GPU partition (`divide` on the fused position variable,
 *     snapped to segments)                  SPEC.md:248-256, SURVEY.md §8(e)
 *   - the value semantics of every kernel in the table, i.e. dense_eval
 *     (tensors.py:300-330) restricted to the stored nonzeros, walking the
 *     coordinate hierarchy exactly as Tensor._walk does (tensors.py:189-205):
 *       SpMV   y(i)   = sum_j A(i,j) x(j)
 *       SpMM   C(i,k) = sum_j A(i,j) B(j,k)
 *       SDDMM  A(i,j) = B(i,j) * sum_k C(i,k) D(j,k)   (on B's pattern)
 *       TTV    A(i,j) = sum_k B(i,j,k) c(k)
 *       MTTKRP A(i,j) = sum_{k,l} B(i,k,l) C(k,j) D(l,j)
 *     accumulating in fp64 over fp32 or fp64 inputs (BASELINE.md §2 parity
 *     rule: oracle in fp64 on the fp32-rounded inputs).
 *
 * The restatement is pinned to the reference by tests/test_oracle.py against
 * golden vectors produced by importing the reference (tests/golden/).
 * OpenMP parallelises over output rows/slices; results do not depend on the
 * thread count (each output row is summed by one thread in position order).
 */
#include <stdint.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

int orc_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ir.py:178-190: largest s in [lo,hi) with arr[s] <= key, clamped */
int64_t orc_search_segment(const int32_t* arr, int64_t lo, int64_t hi, int64_t key) {
  if (hi <= lo) return lo;
  int64_t a = lo, b = hi;
  while (a < b) {
    int64_t mid = a + (b - a) / 2;
    if ((int64_t)arr[mid] <= key) a = mid + 1;
    else b = mid;
  }
  return a - 1 < lo ? lo : a - 1;
}

/* ir.py:193-205: first s in [lo,hi) with arr[s] >= key, else hi */
int64_t orc_search_coord(const int32_t* arr, int64_t lo, int64_t hi, int64_t key) {
  for (int64_t s = lo; s < hi; ++s)
    if ((int64_t)arr[s] >= key) return s;
  return hi;
}

/* R_g = first s with seg_start[s] >= min(g*ceil(nnz/G), nnz) */
int orc_partition(const int32_t* seg_start, int64_t nseg, int64_t nnz, int32_t ndev, int64_t* out) {
  if (ndev < 1) return 1;
  int64_t chunk = (nnz + ndev - 1) / ndev;
  out[0] = 0;
  for (int g = 1; g < ndev; ++g) {
    int64_t t = (int64_t)g * chunk;
    if (t > nnz) t = nnz;
    out[g] = orc_search_coord(seg_start, 0, nseg, t);
  }
  out[ndev] = nseg;
  return 0;
}

#define VAL(p, k) (is_f32 ? (double)((const float*)(p))[k] : ((const double*)(p))[k])

/* SpMV over CSR ("ds"): pos/crd of level 1 */
void orc_spmv(int64_t M, const int32_t* pos, const int32_t* crd, const void* vals, const void* x, int is_f32,
              double* y) {
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t i = 0; i < M; ++i) {
    double acc = 0.0;
    for (int64_t p = pos[i]; p < pos[i + 1]; ++p) acc += VAL(vals, p) * VAL(x, crd[p]);
    y[i] = acc;
  }
}

/* SpMM: C[M x N] = A[M x K] (CSR) * B[K x N] (row-major).  Rows [r0, r1). */
void orc_spmm_rows(int64_t r0, int64_t r1, int64_t N, const int32_t* pos, const int32_t* crd, const void* vals,
                   const void* B, int is_f32, double* C) {
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t i = r0; i < r1; ++i) {
    double* c = C + (i - r0) * N;
    for (int64_t k = 0; k < N; ++k) c[k] = 0.0;
    for (int64_t p = pos[i]; p < pos[i + 1]; ++p) {
      const double a = VAL(vals, p);
      const int64_t j = crd[p];
      if (is_f32) {
        const float* b = (const float*)B + j * N;
        for (int64_t k = 0; k < N; ++k) c[k] += a * (double)b[k];
      } else {
        const double* b = (const double*)B + j * N;
        for (int64_t k = 0; k < N; ++k) c[k] += a * b[k];
      }
    }
  }
}

void orc_spmm(int64_t M, int64_t N, const int32_t* pos, const int32_t* crd, const void* vals, const void* B,
              int is_f32, double* C) {
  orc_spmm_rows(0, M, N, pos, crd, vals, B, is_f32, C);
}

/* SDDMM on B's pattern: out[p] = Bv[p] * <C[i,:], D[crd[p],:]> */
void orc_sddmm(int64_t M, int64_t K, const int32_t* pos, const int32_t* crd, const void* vals, const void* Cm,
               const void* Dm, int is_f32, double* out) {
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t i = 0; i < M; ++i) {
    for (int64_t p = pos[i]; p < pos[i + 1]; ++p) {
      const int64_t j = crd[p];
      double s = 0.0;
      for (int64_t k = 0; k < K; ++k) s += VAL(Cm, i * K + k) * VAL(Dm, j * K + k);
      out[p] = VAL(vals, p) * s;
    }
  }
}

/* TTV on CSF ("sss"): A[I x J] dense, zero where no fiber */
void orc_ttv(int64_t S, int64_t J, const int32_t* crd0, const int32_t* pos1, const int32_t* crd1,
             const int32_t* pos2, const int32_t* crd2, const void* vals, const void* c, int is_f32, double* A,
             int64_t I) {
  memset(A, 0, sizeof(double) * (size_t)(I * J));
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t s = 0; s < S; ++s) {
    const int64_t i = crd0[s];
    for (int64_t f = pos1[s]; f < pos1[s + 1]; ++f) {
      double acc = 0.0;
      for (int64_t p = pos2[f]; p < pos2[f + 1]; ++p) acc += VAL(vals, p) * VAL(c, crd2[p]);
      A[i * J + crd1[f]] = acc;
    }
  }
}

/* MTTKRP on CSF: A[I x R] = sum B(i,k,l) C(k,:) * D(l,:) */
void orc_mttkrp(int64_t S, int64_t R, const int32_t* crd0, const int32_t* pos1, const int32_t* crd1,
                const int32_t* pos2, const int32_t* crd2, const void* vals, const void* Cm, const void* Dm,
                int is_f32, double* A, int64_t I) {
  memset(A, 0, sizeof(double) * (size_t)(I * R));
#pragma omp parallel
  {
    double* fib = (double*)__builtin_alloca(sizeof(double) * (size_t)R);
#pragma omp for schedule(dynamic, 1)
    for (int64_t s = 0; s < S; ++s) {
      double* a = A + (int64_t)crd0[s] * R;
      for (int64_t f = pos1[s]; f < pos1[s + 1]; ++f) {
        for (int64_t r = 0; r < R; ++r) fib[r] = 0.0;
        for (int64_t p = pos2[f]; p < pos2[f + 1]; ++p) {
          const double v = VAL(vals, p);
          const int64_t l = crd2[p];
          for (int64_t r = 0; r < R; ++r) fib[r] += v * VAL(Dm, l * R + r);
        }
        const int64_t k = crd1[f];
        for (int64_t r = 0; r < R; ++r) a[r] += fib[r] * VAL(Cm, k * R + r);
      }
    }
  }
}
