// batchlp/batchlp.hpp — umbrella header of the B200 drop-in.
//
// Covers the reference's umbrella (reference proj/include/batchlp/
// batchlp.hpp:18-29) except the instance generators and the test-only
// vertex-enumeration oracle (out of scope): the hot
// path, the drivers, the device batch-width tuner, MPS I/O and -- when
// nlohmann/json is on the include path, as the reference requires -- the
// JSON reports. Link with -lbatchlp_cuda
// (paper_2601_21990_b200/lib/).
#ifndef BATCHLP_B200_BATCHLP_HPP
#define BATCHLP_B200_BATCHLP_HPP

#include "batchlp/batch_solver.hpp"
#include "batchlp/bounds.hpp"
#include "batchlp/mps.hpp"
#include "batchlp/obbt.hpp"
#include "batchlp/problem.hpp"
#include "batchlp/solver.hpp"
#include "batchlp/sparse.hpp"
#include "batchlp/strong_branching.hpp"
#include "batchlp/tuner.hpp"
#if __has_include(<nlohmann/json.hpp>)
#include "batchlp/report.hpp"
#endif

#endif  // BATCHLP_B200_BATCHLP_HPP
