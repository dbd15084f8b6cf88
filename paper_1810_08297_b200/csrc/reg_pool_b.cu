// Registration group: the second half of the reference test-suite kernel
// pool (reg_pool.cu; proj/tests/support/kernel_pool.hpp:19-102).
#include "bodies.cuh"
#include "launch.cuh"

static const bcad_cu_kernel_entry kEntries[] = {
    BCAD_ENTRY(bcad_dev::KCurl),     BCAD_ENTRY(bcad_dev::KFanout),     BCAD_ENTRY(bcad_dev::KFiveway),
    BCAD_ENTRY(bcad_dev::KWave),     BCAD_ENTRY(bcad_dev::KGate),       BCAD_ENTRY(bcad_dev::KSigTanh),
    BCAD_ENTRY(bcad_dev::KSquareGate), BCAD_ENTRY(bcad_dev::KTwo),      BCAD_ENTRY(bcad_dev::KExp),
};

int bcad_reg_pool_b(const bcad_cu_kernel_entry** out) {
    *out = kEntries;
    return int(sizeof(kEntries) / sizeof(kEntries[0]));
}
