// Umbrella header of the drop-in C++ API (mirrors
// /root/reference/proj/include/parafac2/parafac2.hpp).  Link with
// paper_1703_04219_b200/lib/libp2g.so.
#pragma once

#include "common.hpp"
#include "cp.hpp"
#include "kernels.hpp"
#include "mttkrp.hpp"
#include "slices.hpp"
#include "solver.hpp"
#include "sparse.hpp"
#include "io.hpp"
