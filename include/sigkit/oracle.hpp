#pragma once
// Drop-in replacement for the reference's brute-force oracle
// (/root/reference/proj/include/sigkit/oracle.hpp:1-35): same types, limits
// and exceptions; the enumeration runs on the GPU (sigk_signature_bruteforce_f64,
// fp64 bit-identical to the reference).

#include <cstddef>
#include <vector>

#include "sigkit/tensor_algebra.hpp"

namespace sigkit {

struct OracleLimits {
    int max_segments = 8;
    int max_depth = 4;
    int max_dim = 3;
};

enum class TupleClass { WeaklyIncreasing, StrictlyIncreasing };

FlatSignature signature_bruteforce(const std::vector<double>& path, std::size_t len, int dim, int depth,
                                   const OracleLimits& limits = OracleLimits{},
                                   TupleClass tuples = TupleClass::WeaklyIncreasing);

}  // namespace sigkit
