# gradient kernel A/Bs (kgrad.cuh knobs); usage: bash tools/gpu_grad.sh
# experiment builds first (CPU):  python -c "from paper_2301_11389_b200 import build as b;
#   b.build_experiment('g_minb6', ('STB200_GRAD_MINB=6',)); b.build_experiment('g_cs', ('STB200_GRAD_CS=1',));
#   b.build_experiment('g_w4', ('STB200_GRAD_WARPS=4',)); b.build_experiment('g_w16', ('STB200_GRAD_WARPS=16',))"
for zc in 4 8 16 32; do echo "== kgrad zc=$zc"; STB200_GRAD_ZC=$zc bash tools/bench_all.sh gradient; done
echo "== k3d"; STB200_GRAD_K3D=1 bash tools/bench_all.sh gradient
for e in g_minb6 g_cs g_w4 g_w16; do
  [ -f expbuild/$e/libstencil_b200.so ] || continue
  echo "== $e"; STB200_LIB=$PWD/expbuild/$e/libstencil_b200.so bash tools/bench_all.sh gradient
done
