// Registration group: the HM-LSTM cell-update bodies (the north-star path).
#include "bodies.cuh"
#include "launch.cuh"

static const bcad_cu_kernel_entry kEntries[] = {
    BCAD_ENTRY(bcad_dev::KHmlstm, bcad_cu_impl::SigHmlstmCanonical, bcad_cu_impl::SigHmlstmDivergence),
    BCAD_ENTRY(bcad_dev::KHmlstmBias, bcad_cu_impl::SigHmlstmBias),
};

int bcad_reg_hmlstm(const bcad_cu_kernel_entry** out) {
    *out = kEntries;
    return int(sizeof(kEntries) / sizeof(kEntries[0]));
}
