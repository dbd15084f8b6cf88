// Device twins of the kernel bodies the reference's own test suites define as
// test-local lambdas (proj/tests/test_broadcast.cpp:109-220,
// test_forward.cpp:156-160). Porting a reference user's lambda body is
// exactly this step: the same expression, written once in an nvcc
// translation unit and registered by name (bcad/device_kernel.cuh); the
// suites' BroadcastKernel(n, m, name, lambda) then binds it and checks the
// lambda against it. Linked into tests/cpp/bin/ref_suites_b200 only.
#include "bcad/device_kernel.cuh"

// test_broadcast.cpp:109-112
BCAD_DEVICE_KERNEL_NOTHROW_P(RefPair, "pair", 3, 2, 0u, out[0] = in[0] * in[1] + in[2];
                             out[1] = tanh(in[0]) - in[2] * in[1])
// test_broadcast.cpp:154-155
BCAD_DEVICE_KERNEL_NOTHROW_P(RefMix, "mix", 2, 1, 0u, out[0] = sigmoid(in[0]) * in[1])
// test_broadcast.cpp:197-198
BCAD_DEVICE_KERNEL_NOTHROW_P(RefWarp, "warp", 1, 1, 0u, out[0] = tanh(in[0]) * in[0])
// test_broadcast.cpp:217-220
BCAD_DEVICE_KERNEL_NOTHROW_P(RefSplit, "split", 1, 2, 0u, out[0] = in[0]; out[1] = -in[0])
// test_forward.cpp:156-160
BCAD_DEVICE_KERNEL_NOTHROW_P(RefOne, "one", 1, 1, 0u, out[0] = tanh(in[0]))
BCAD_DEVICE_KERNEL_NOTHROW_P(RefThree, "three", 3, 2, 0u, out[0] = in[0] * in[1] + in[2]; out[1] = in[0] - in[2])
