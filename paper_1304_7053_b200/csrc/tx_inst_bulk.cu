// Size-specialised bulk (TMA) instances for one scalar type and one op(A):
// every square n = 1..16, every op(B), beta == 0 and general epilogues
// (compile-time polymorphism in the spirit of PAPER.md:414-421).
#include "tx_types.cuh"

#ifndef TX_OPA
#error "TX_OPA must be 0..2"
#endif

namespace tx {
void TX_CAT(TX_CAT(TX_CAT(register_bulk_, TX_T), _), TX_OPA)(TypeTables &t)
{
    using Seq = std::make_integer_sequence<int, 16>;
    fill_square<TxT, TX_OPA, OP_N, false>(t, Seq{});
    fill_square<TxT, TX_OPA, OP_N, true>(t, Seq{});
    fill_square<TxT, TX_OPA, OP_T, false>(t, Seq{});
    fill_square<TxT, TX_OPA, OP_T, true>(t, Seq{});
#if TX_T >= 2
    fill_square<TxT, TX_OPA, OP_C, false>(t, Seq{});
    fill_square<TxT, TX_OPA, OP_C, true>(t, Seq{});
#endif
}
}  // namespace tx
