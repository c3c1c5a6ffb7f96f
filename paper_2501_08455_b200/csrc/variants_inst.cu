// One (precision, d) row of the variant table. Compiled once per pair with
//   -DSIGK_REAL=float|double -DSIGK_DIM=<d>   (see paper_2501_08455_b200/build.py)
#include "variants.cuh"

#ifndef SIGK_REAL
#error "SIGK_REAL must be defined"
#endif
#ifndef SIGK_DIM
#error "SIGK_DIM must be defined"
#endif

#define SIGK_CAT_(a, b) a##b
#define SIGK_CAT(a, b) SIGK_CAT_(a, b)

namespace sigk {
namespace {
using Row = DimTable<SIGK_REAL, SIGK_DIM, SIGK_CAT(SIGK_DEPTHS_, SIGK_DIM)>;
struct Registrar {
    Registrar() { register_variants(Row::table(), Row::count, sizeof(SIGK_REAL) == 8); }
};
Registrar registrar;
}  // namespace
}  // namespace sigk
