// snp_tiled.cu -- instances of tiled_step_kernel (snp_device.cuh) for one P
// mode, selected with -DSNP_TILED_PM=<0..3>; build.py compiles the four
// objects in parallel and links them with snp_engine.cu.
#define SNP_TEMPLATES_ONLY
#include "snp_device.cuh"

#ifndef SNP_TILED_PM
#error "compile with -DSNP_TILED_PM=<P mode>"
#endif

namespace snp {

namespace {
template <int PM, int RW>
void pick_cb(int cb, TiledFn* step, TiledFn* lean) {
    switch (cb) {
        case 8:
            *step = tiled_step_kernel<PM, RW, 8, false>;
            *lean = tiled_step_kernel<PM, RW, 8, true>;
            break;
        case 16:
            *step = tiled_step_kernel<PM, RW, 16, false>;
            *lean = tiled_step_kernel<PM, RW, 16, true>;
            break;
        default:
            *step = tiled_step_kernel<PM, RW, 32, false>;
            *lean = tiled_step_kernel<PM, RW, 32, true>;
    }
}
}  // namespace

template <>
void tiled_fns<SNP_TILED_PM>(int rw, int cb, TiledFn* step, TiledFn* lean) {
    if (rw == RW_WIDE) pick_cb<SNP_TILED_PM, RW_WIDE>(cb, step, lean);
    else if (rw == RW_TINY) pick_cb<SNP_TILED_PM, RW_TINY>(cb, step, lean);
    else pick_cb<SNP_TILED_PM, RW_COMPACT>(cb, step, lean);
}

}  // namespace snp
