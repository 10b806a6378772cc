// Generic-size instances for one scalar type: bulk kernels for any packed
// m, n, k <= 16, gather kernels (general strided and pointer-array layouts),
// and the alpha == 0 / k == 0 scale kernels.
#include "tx_types.cuh"
#include "tx_tc.cuh"

namespace tx {
namespace {
template <int OPA, int OPB>
void fill_ops(TypeTables &t)
{
    t.bulk_dyn[OPA][OPB][0] = &launch_bulk<TxT, 0, 0, 0, OPA, OPB, false>;
    t.bulk_dyn[OPA][OPB][1] = &launch_bulk<TxT, 0, 0, 0, OPA, OPB, true>;
    t.gather[OPA][OPB][0][0] = &launch_gather<TxT, OPA, OPB, false, false>;
    t.gather[OPA][OPB][1][0] = &launch_gather<TxT, OPA, OPB, true, false>;
    t.gather[OPA][OPB][0][1] = &launch_gather<TxT, OPA, OPB, false, true>;
    t.gather[OPA][OPB][1][1] = &launch_gather<TxT, OPA, OPB, true, true>;
    t.bulk_dyn_dev[OPA][OPB] = &launch_bulk_dev<TxT, OPA, OPB>;
    t.gather_dev[OPA][OPB][0] = &launch_gather_dev<TxT, OPA, OPB, false>;
    t.gather_dev[OPA][OPB][1] = &launch_gather_dev<TxT, OPA, OPB, true>;
    t.direct[OPA][OPB][0][0] = &launch_direct<TxT, 1, OPA, OPB, false>;
    t.direct[OPA][OPB][1][0] = &launch_direct<TxT, 1, OPA, OPB, true>;
    t.direct[OPA][OPB][0][1] = &launch_direct<TxT, 2, OPA, OPB, false>;
    t.direct[OPA][OPB][1][1] = &launch_direct<TxT, 2, OPA, OPB, true>;
    t.count += 13;
    if constexpr (TcOk<TxT>::value) {
        t.tc[OPA][OPB][0] = &launch_tc<TxT, OPA, OPB, false>;
        t.tc[OPA][OPB][1] = &launch_tc<TxT, OPA, OPB, true>;
        t.count += 2;
    }
}
}  // namespace

void TX_CAT(register_gen_, TX_T)(TypeTables &t)
{
    fill_ops<OP_N, OP_N>(t);
    fill_ops<OP_N, OP_T>(t);
    fill_ops<OP_T, OP_N>(t);
    fill_ops<OP_T, OP_T>(t);
#if TX_T >= 2
    fill_ops<OP_N, OP_C>(t);
    fill_ops<OP_T, OP_C>(t);
    fill_ops<OP_C, OP_N>(t);
    fill_ops<OP_C, OP_T>(t);
    fill_ops<OP_C, OP_C>(t);
#endif
    t.scale[0][0] = &launch_scale<TxT, false, false>;
    t.scale[0][1] = &launch_scale<TxT, false, true>;
    t.scale[1][0] = &launch_scale<TxT, true, false>;
    t.scale[1][1] = &launch_scale<TxT, true, true>;
    t.scale_dev[0] = &launch_scale<TxT, false, false, true>;
    t.scale_dev[1] = &launch_scale<TxT, true, false, true>;
    t.count += 6;
}
}  // namespace tx
