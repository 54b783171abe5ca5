# gradient kernel A/Bs (kgrad.cuh knobs); usage: bash tools/gpu_grad.sh
for zc in 4 6 8; do echo "== base zc=$zc"; STB200_GRAD_ZC=$zc bash tools/bench_all.sh gradient; done
for e in g_w4 g_w16; do for zc in 6 8; do echo "== $e zc=$zc"; STB200_LIB=$PWD/expbuild/$e/libstencil_b200.so STB200_GRAD_ZC=$zc bash tools/bench_all.sh gradient; done; done
