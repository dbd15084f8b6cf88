// Registration group: bodies whose dual rules can raise (error-path probes:
// dual.hpp:129-166 division, 284-342 log/sqrt/abs/pow domains).
#include "bodies.cuh"
#include "launch.cuh"

static const bcad_cu_kernel_entry kEntries[] = {
    BCAD_ENTRY(bcad_dev::KLog), BCAD_ENTRY(bcad_dev::KDiv), BCAD_ENTRY(bcad_dev::KSqrt), BCAD_ENTRY(bcad_dev::KAbs), BCAD_ENTRY(bcad_dev::KPowHalf), BCAD_ENTRY(bcad_dev::KRecip),
};

int bcad_reg_probe(const bcad_cu_kernel_entry** out) {
    *out = kEntries;
    return int(sizeof(kEntries) / sizeof(kEntries[0]));
}
