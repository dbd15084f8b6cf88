// Registration group: tensor-level tape primitives (reference
// proj/include/bcad/tape.hpp:84-129 forward values, 284-330 backward rules).
#include "bodies.cuh"
#include "launch.cuh"

static const bcad_cu_kernel_entry kEntries[] = {
    BCAD_ENTRY(bcad_dev::KMinus),       BCAD_ENTRY(bcad_dev::KNeg),           BCAD_ENTRY(bcad_dev::KSigmoid),
    BCAD_ENTRY(bcad_dev::KTanh),        BCAD_ENTRY(bcad_dev::KSelect),        BCAD_ENTRY(bcad_dev::KSigmoidBwd),
    BCAD_ENTRY(bcad_dev::KTanhBwd),     BCAD_ENTRY(bcad_dev::KSelectTrueBwd), BCAD_ENTRY(bcad_dev::KSelectFalseBwd),
};

int bcad_reg_prims(const bcad_cu_kernel_entry** out) {
    *out = kEntries;
    return int(sizeof(kEntries) / sizeof(kEntries[0]));
}
