// Registration group: the reference test-suite kernel pool
// (proj/tests/support/kernel_pool.hpp:19-102, test_mixed.cpp, test_broadcast.cpp).
#include "bodies.cuh"
#include "launch.cuh"

// (split over two translation units, reg_pool_b.cu, which compile in parallel)
static const bcad_cu_kernel_entry kEntries[] = {
    BCAD_ENTRY(bcad_dev::KIdentity), BCAD_ENTRY(bcad_dev::KReflect), BCAD_ENTRY(bcad_dev::KTanhSigmoid),
    BCAD_ENTRY(bcad_dev::KProduct),  BCAD_ENTRY(bcad_dev::KMul),     BCAD_ENTRY(bcad_dev::KPlus),
    BCAD_ENTRY(bcad_dev::KGated),    BCAD_ENTRY(bcad_dev::KProdDiff), BCAD_ENTRY(bcad_dev::KBlend),
};

int bcad_reg_pool(const bcad_cu_kernel_entry** out) {
    *out = kEntries;
    return int(sizeof(kEntries) / sizeof(kEntries[0]));
}
