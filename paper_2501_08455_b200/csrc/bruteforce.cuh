// Brute-force signature of one path by direct enumeration of segment-index
// tuples (reference signature_bruteforce, oracle.cpp:28-96): the ground-truth
// oracle of the reference's own tests, part of its public API. One thread per
// output coefficient walks the tuples in the reference's odometer order with
// the same products (left-associated tensor products, then weight * term,
// then the sum, no contraction into FMAs), so fp64 results are bit-identical.
#pragma once
#include <cstdint>

namespace sigk {

constexpr int kBruteMaxDepth = 8;

__global__ void bruteforce_kernel(const double* __restrict__ path, int segments, int d, int depth, int strict,
                                  double* __restrict__ out) {
    // coefficient q: level n, flat index idx (last index fastest)
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int n = 1;
    int64_t size = d, off = 0;
    while (n <= depth && q >= off + size) {
        off += size;
        size *= d;
        ++n;
    }
    if (n > depth) return;
    const int64_t idx = q - off;
    int dig[kBruteMaxDepth];
    {
        int64_t r = idx;
        for (int k = n - 1; k >= 0; --k) {
            dig[k] = (int)(r % d);
            r /= d;
        }
    }
    double acc = 0.0;
    if (segments > 0 && !(strict && n > segments)) {
        int tup[kBruteMaxDepth];
        for (int i = 0; i < n; ++i) tup[i] = strict ? i : 0;
        while (true) {
            double term = path[(int64_t)(tup[0] + 1) * d + dig[0]] - path[(int64_t)tup[0] * d + dig[0]];
            for (int i = 1; i < n; ++i)
                term = __dmul_rn(term, path[(int64_t)(tup[i] + 1) * d + dig[i]] - path[(int64_t)tup[i] * d + dig[i]]);
            double w = 1.0;
            if (!strict) {  // 1 / product over runs of equal indices of (run length)!
                double denom = 1.0;
                int run = 1;
                for (int i = 1; i < n; ++i) {
                    if (tup[i] == tup[i - 1]) {
                        ++run;
                        denom = __dmul_rn(denom, (double)run);
                    } else {
                        run = 1;
                    }
                }
                w = 1.0 / denom;
            }
            acc = __dadd_rn(acc, __dmul_rn(w, term));
            int pos = n - 1;
            while (pos >= 0 && tup[pos] == segments - 1 - (strict ? (n - 1 - pos) : 0)) --pos;
            if (pos < 0) break;
            ++tup[pos];
            for (int i = pos + 1; i < n; ++i) tup[i] = tup[i - 1] + (strict ? 1 : 0);
        }
    }
    out[q] = acc;
}

}  // namespace sigk
