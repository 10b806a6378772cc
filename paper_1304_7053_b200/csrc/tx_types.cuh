// tx_types.cuh -- compile-time selection of the scalar type for an
// instantiation unit (-DTX_T=0..3) and token pasting helpers.
#pragma once
#include "tx_dispatch.cuh"

#define TX_CAT_(a, b) a##b
#define TX_CAT(a, b) TX_CAT_(a, b)

#if TX_T == 0
using TxT = float;
#elif TX_T == 1
using TxT = double;
#elif TX_T == 2
using TxT = float2;
#elif TX_T == 3
using TxT = double2;
#else
#error "TX_T must be 0..3"
#endif
