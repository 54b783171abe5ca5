bash tools/gpu_flake_all.sh > gpurun_out/flake_all.txt 2>&1; cat gpurun_out/flake_all.txt
bash tools/bench_all.sh gaussblur jacobi2d_paper gameoflife laplacian wave13pt jacobi3d divergence tricubic > gpurun_out/bench_rel1.txt 2>&1
STB200_LIB=expbuild/rel2/libstencil_b200.so bash tools/bench_all.sh gaussblur jacobi2d_paper gameoflife laplacian wave13pt jacobi3d divergence tricubic > gpurun_out/bench_rel2.txt 2>&1
paste gpurun_out/bench_rel1.txt gpurun_out/bench_rel2.txt | awk '{print $1, $2, $3, "vs", $(NF/2+3)}'
