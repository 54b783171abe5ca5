for b in 0 1; do echo "BULK=$b"; STB200_BULK=$b bash tools/bench_all.sh laplacian wave13pt jacobi3d gradient; done
