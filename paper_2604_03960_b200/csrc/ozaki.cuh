// Emulated-FP64 GEMM on the int8 tensor cores (Ozaki scheme, tcgen05.mma
// kind::i8); see ozaki.cu.
#pragma once

#include "common.cuh"

namespace achi {

constexpr int OZ_MAX_SLICES = 9;

// C (M x N, row-major, ldc) = A B in emulated FP64 with `slices` 7-bit digits per
// operand entry (s = 8: 56 bits, FP64-level; fewer: faster, less accurate).
// A: M x K row-major (lda), or K x M row-major when a_trans.  B: K x N row-major
// (ldb), or N x K row-major when b_kmajor.  K <= 16384.
// Workspace: ctx.oz_digits (int8 digit planes), ctx.oz_ex (exponents).
void dgemm_ozaki(Ctx& ctx, int M, int N, int K, const double* A, long lda, bool a_trans,
                 const double* B, long ldb, bool b_kmajor, double* C, long ldc, int slices);

}  // namespace achi
