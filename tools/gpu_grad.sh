# gradient kernel A/Bs (kgrad.cuh knobs); usage: bash tools/gpu_grad.sh
STB200_GRAD_RPW=2 timeout 600 python -m pytest tests -q -m gpu -k "gradient" 2>&1 | tail -1
echo "== kgrad zc=8"; bash tools/bench_all.sh gradient
for zc in 8 16; do echo "== kgrad2 minb3 zc=$zc"; STB200_GRAD_RPW=2 STB200_GRAD_ZC=$zc bash tools/bench_all.sh gradient; done
for e in g2_minb4 g2_minb2; do echo "== $e zc=8"; STB200_LIB=$PWD/expbuild/$e/libstencil_b200.so STB200_GRAD_RPW=2 STB200_GRAD_ZC=8 bash tools/bench_all.sh gradient; done
