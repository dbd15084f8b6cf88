// Registration group: the reference test-suite kernel pool
// (proj/tests/support/kernel_pool.hpp:19-102, test_mixed.cpp, test_broadcast.cpp).
#include "bodies.cuh"
#include "launch.cuh"

static const bcad_cu_kernel_entry kEntries[] = {
    BCAD_ENTRY(bcad_dev::KIdentity),   BCAD_ENTRY(bcad_dev::KReflect), BCAD_ENTRY(bcad_dev::KTanhSigmoid), BCAD_ENTRY(bcad_dev::KProduct),
    BCAD_ENTRY(bcad_dev::KMul),        BCAD_ENTRY(bcad_dev::KPlus),    BCAD_ENTRY(bcad_dev::KGated),       BCAD_ENTRY(bcad_dev::KProdDiff),
    BCAD_ENTRY(bcad_dev::KBlend),      BCAD_ENTRY(bcad_dev::KCurl),    BCAD_ENTRY(bcad_dev::KFanout),      BCAD_ENTRY(bcad_dev::KFiveway),
    BCAD_ENTRY(bcad_dev::KWave),       BCAD_ENTRY(bcad_dev::KGate),    BCAD_ENTRY(bcad_dev::KSigTanh),     BCAD_ENTRY(bcad_dev::KSquareGate),
    BCAD_ENTRY(bcad_dev::KTwo),        BCAD_ENTRY(bcad_dev::KExp),
};

int bcad_reg_pool(const bcad_cu_kernel_entry** out) {
    *out = kEntries;
    return int(sizeof(kEntries) / sizeof(kEntries[0]));
}
