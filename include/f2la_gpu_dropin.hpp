// f2la_gpu_dropin.hpp — opt-in drop-in: the reference's own f2la:: call sites
// run on the B200.
//
// Include this header IN PLACE OF "f2la/m4rm.hpp" (after "f2la/bit_matrix.hpp").
// It claims the reference header's include guard (F2LA_M4RM_HPP, m4rm.hpp:1-2),
// so a later #include "f2la/m4rm.hpp" is a no-op, and it declares the names that
// header defines -- M4rmTables, make_splits, build_tables (4 overloads),
// mult_acc, m4rm_mult (m4rm.hpp:21-196) -- in namespace f2la as the GPU-backed
// versions of include/f2la_gpu.hpp.  The SPEC-declared entry points the
// reference leaves to its users (strassen_mult, decompose_block,
// decompose_recursive, rank, null_space, solve) are brought in
// too.  Code written against the reference, e.g. a Schur-update loop
//
//     auto splits = f2la::make_splits(k, c);
//     auto t = f2la::build_tables(b, row0, k, wcol0, n, std::span<const std::uint32_t>(splits));
//     f2la::mult_acc(c_mat, c_row0, c_wcol0, a_words, t);
//
// compiles unchanged and executes on the device (libf2gpu.so).
//
// One translation unit sees either the CPU or the GPU definitions, never both:
// do not mix this header with "f2la/m4rm.hpp" templates instantiated in other
// translation units of the same program (ODR).  Only Word = std::uint64_t.
#ifndef F2LA_GPU_DROPIN_HPP
#define F2LA_GPU_DROPIN_HPP

#ifdef F2LA_M4RM_HPP
#error "f2la_gpu_dropin.hpp must be included instead of (not after) f2la/m4rm.hpp"
#endif
#define F2LA_M4RM_HPP

#include "f2la/bit_matrix.hpp"
#include "f2la/tuning.hpp"
#include "f2la_gpu.hpp"

namespace f2la {

template <WordType Word>
using M4rmTables = gpu::M4rmTables<Word>;

using gpu::build_tables;
using gpu::decompose_block;
using gpu::decompose_recursive;
using gpu::m4rm_mult;
using gpu::make_splits;
using gpu::mult_acc;
using gpu::null_space;
using gpu::rank;
using gpu::solve;
using gpu::strassen_mult;

}  // namespace f2la

#endif
