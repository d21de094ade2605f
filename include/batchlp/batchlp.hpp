// batchlp/batchlp.hpp — umbrella header of the B200 drop-in.
//
// Covers the hot-path subset of the reference's umbrella
// (reference proj/include/batchlp/batchlp.hpp:18-29) plus the device batch-
// width tuner: generators, MPS I/O, JSON reports and
// the vertex-enumeration oracle are out of scope and
// are not declared here. Link with
// -lbatchlp_cuda (paper_2601_21990_b200/lib/).
#ifndef BATCHLP_B200_BATCHLP_HPP
#define BATCHLP_B200_BATCHLP_HPP

#include "batchlp/batch_solver.hpp"
#include "batchlp/bounds.hpp"
#include "batchlp/obbt.hpp"
#include "batchlp/problem.hpp"
#include "batchlp/solver.hpp"
#include "batchlp/sparse.hpp"
#include "batchlp/strong_branching.hpp"
#include "batchlp/tuner.hpp"

#endif  // BATCHLP_B200_BATCHLP_HPP
