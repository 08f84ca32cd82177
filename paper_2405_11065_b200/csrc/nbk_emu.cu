// nbk_emu.cu -- precision-emulated solves: the CG loop of
// enqueue_solve instantiated with PM = NBK_EMU_MODE (compiled once per mode by
// build.py, -DNBK_EMU_MODE=1/2/3, in parallel).  Entry points are suffixed by
// the mode; enqueue_emulated / emulated_attrs in nbk_capi.cu select them.
#include "nbk_launch.cuh"

namespace nbk {

#define NBK_EMU_CAT2(a, b) a##b
#define NBK_EMU_CAT(a, b) NBK_EMU_CAT2(a, b)

cudaError_t NBK_EMU_CAT(enqueue_emulated_, NBK_EMU_MODE)(const Team& t, int niter, nbk_graph* g,
                                                         bool profiling, std::string& err)
{
    return enqueue_solve<double, NBK_EMU_MODE>(t, niter, g, false, profiling, err);
}

cudaError_t NBK_EMU_CAT(emulated_attrs_, NBK_EMU_MODE)(nbk_ctx* c)
{
    if (NBK_EMU_MODE != PM_VPREC && c->N > NBK_MC_MAXN) return cudaSuccess;
    AxArgs<double> a64{};
    a64.mesh = c->view;
    cudaError_t e = dssum_attrs<double, true, NBK_EMU_MODE>();
    if (e != cudaSuccess) return e;
    return launch_ax<double, 1, NBK_EMU_MODE>(a64, c->stream, true);
}

}  // namespace nbk
