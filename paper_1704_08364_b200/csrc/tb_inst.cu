// tb_inst.cu -- instantiates the launchers (and with them every kernel
// template) for one radial length L = TB_L; compiled once per L.
#include "tb_launch.cuh"

#ifndef TB_L
#error "compile with -DTB_L=<radial length>"
#endif

#define TB_CAT2(a, b) a##b
#define TB_CAT(a, b) TB_CAT2(a, b)

int TB_CAT(tb_configure_, TB_L)(tb_plan* p) { return Launch<TB_L>::configure(p); }

int TB_CAT(tb_group_, TB_L)(const tb_plan* p, const float* sino, float* img, int B, const Work& w, bool ramp,
                            float scale, cudaStream_t st, cudaEvent_t* ev) {
  return Launch<TB_L>::bst_group(p, sino, img, B, w, ramp, scale, st, ev);
}

int TB_CAT(tb_ramp_, TB_L)(const tb_plan* p, const float* in, float* out, int total_rows, const Work& w,
                           cudaStream_t st) {
  return launch_ramp<TB_L>(p, in, out, total_rows, w, st);
}

int TB_CAT(tb_pipe_, TB_L)(const tb_plan* p, const float* sino, float* img, int n_slices, int batch,
                           const Work* lanes, size_t in_stride, size_t out_stride, float scale, bool with_k3,
                           cudaStream_t st) {
  return Launch<TB_L>::fused_pipeline(p, sino, img, n_slices, batch, lanes, in_stride, out_stride, scale, with_k3,
                                      st);
}
