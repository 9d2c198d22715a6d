/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously correct CPU reference for y = A*x with A in CRS.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may load this
 * library.  It shares no code, header or constant with paper_1112_5588_b200/ (the CUDA path).
 *
 * Definition followed (§1.1 "spMVM ... y = A x"; Table 1 "CRS (DP)";
 * SPEC.md L206-209 spmv_csr):   y_i = sum_{k = rowptr[i]}^{rowptr[i+1]-1} val[k] * x[col[k]].
 *
 * Functions:
 *   oracle_spmv_ld      O1: long double (x86 80-bit) products and accumulation of the
 *                       stored values, plus bound_i = sum_k |val[k] x[col[k]]|.
 *   oracle_spmv_chain   O3: one fused-multiply-add chain per row in stored CRS order, starting
 *                       from +0.0, in the matrix precision (reading 14).
 *   oracle_spmv_crs     the plain CRS loop in the target precision (DP: double, SP: float
 *                       accumulation), OpenMP static over rows: the CPU baseline that is timed
 *                       (Table 1 "Westmere EP CRS (DP)").
 * Compiled with -ffp-contract=off so that every a*b+c is exactly what the source says.
 */
#include <math.h>
#include <stdint.h>
#include <omp.h>

/* dtype: 0 = float32 values/x, 1 = float64 values/x */

void oracle_spmv_ld(int64_t n, const int64_t* rowptr, const int32_t* col, const void* val,
                    const void* x, int dtype, long double* y, long double* bound) {
  /* Rows are independent, so threading over rows changes nothing in any y_i. */
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    long double s = 0.0L, b = 0.0L;
    for (int64_t k = rowptr[i]; k < rowptr[i + 1]; ++k) {
      long double a, xv;
      if (dtype == 1) {
        a = ((const double*)val)[k];
        xv = ((const double*)x)[col[k]];
      } else {
        a = ((const float*)val)[k];
        xv = ((const float*)x)[col[k]];
      }
      long double p = a * xv; /* SP: exact (24x24 bits); DP: relative error <= 2^-64 */
      s += p;
      b += fabsl(p);
    }
    y[i] = s;
    bound[i] = b;
  }
}

void oracle_spmv_chain(int64_t n, const int64_t* rowptr, const int32_t* col, const void* val,
                       const void* x, int dtype, void* y) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    if (dtype == 1) {
      const double* v = (const double*)val;
      const double* xv = (const double*)x;
      double acc = 0.0;
      for (int64_t k = rowptr[i]; k < rowptr[i + 1]; ++k) acc = fma(v[k], xv[col[k]], acc);
      ((double*)y)[i] = acc;
    } else {
      const float* v = (const float*)val;
      const float* xv = (const float*)x;
      float acc = 0.0f;
      for (int64_t k = rowptr[i]; k < rowptr[i + 1]; ++k) acc = fmaf(v[k], xv[col[k]], acc);
      ((float*)y)[i] = acc;
    }
  }
}

/* The long-row ("split-j") kernel variant's arithmetic (SURVEY §8(c) O3 exemption for split-j
 * kernels; NEXT-4): for S threads per row, partial p_s = fma chain from +0.0 over the row's stored
 * entries with position j = s, s+S, s+2S, ... (CRS order), then the pairwise tree
 * ((p_0+p_1)+(p_2+p_3))+... over s = 0..S-1 (S a power of two).  S = 1 is oracle_spmv_chain. */
void oracle_spmv_split_chain(int64_t n, const int64_t* rowptr, const int32_t* col, const void* val,
                             const void* x, int dtype, int S, void* y) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    double pd[64];
    float pf[64];
    const int64_t r0 = rowptr[i], len = rowptr[i + 1] - rowptr[i];
    for (int s = 0; s < S; ++s) {
      if (dtype == 1) {
        double acc = 0.0;
        for (int64_t j = s; j < len; j += S)
          acc = fma(((const double*)val)[r0 + j], ((const double*)x)[col[r0 + j]], acc);
        pd[s] = acc;
      } else {
        float acc = 0.0f;
        for (int64_t j = s; j < len; j += S)
          acc = fmaf(((const float*)val)[r0 + j], ((const float*)x)[col[r0 + j]], acc);
        pf[s] = acc;
      }
    }
    for (int w = 1; w < S; w *= 2)  /* level w: p_s += p_{s+w} for s a multiple of 2w */
      for (int s = 0; s + w < S; s += 2 * w) {
        if (dtype == 1) pd[s] = pd[s] + pd[s + w];
        else pf[s] = pf[s] + pf[s + w];
      }
    if (dtype == 1) ((double*)y)[i] = pd[0];
    else ((float*)y)[i] = pf[0];
  }
}

void oracle_spmv_crs(int64_t n, const int64_t* rowptr, const int32_t* col, const void* val,
                     const void* x, int dtype, void* y, int nthreads) {
  if (nthreads > 0) omp_set_num_threads(nthreads);
  if (dtype == 1) {
    const double* v = (const double*)val;
    const double* xv = (const double*)x;
    double* yv = (double*)y;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
      double s = 0.0;
      for (int64_t k = rowptr[i]; k < rowptr[i + 1]; ++k) s += v[k] * xv[col[k]];
      yv[i] = s;
    }
  } else {
    const float* v = (const float*)val;
    const float* xv = (const float*)x;
    float* yv = (float*)y;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
      float s = 0.0f;
      for (int64_t k = rowptr[i]; k < rowptr[i + 1]; ++k) s += v[k] * xv[col[k]];
      yv[i] = s;
    }
  }
}

int oracle_max_threads(void) { return omp_get_max_threads(); }
