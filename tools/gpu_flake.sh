# race hunt (tools/flake_hunt.py): the in-tree library vs the plain-arrive build (rel0)
for e in base rel0; do
  if [ $e = base ]; then unset STB200_LIB; else export STB200_LIB=$PWD/expbuild/$e/libstencil_b200.so; fi
  echo "== $e"
  timeout 300 python tools/flake_hunt.py --reps 20 2>&1 | tail -1
  timeout 300 python tools/flake_hunt.py --reps 12 --kind jacobi2d5 --n 16384 --iters 30 2>&1 | tail -1
  timeout 300 python tools/flake_hunt.py --reps 12 --kind gameoflife --dtype i32 --n 16384 --iters 10 2>&1 | tail -1
  timeout 300 python tools/flake_hunt.py --reps 12 --kind laplacian3d7 --dtype f64 --shape 512,512,512 --iters 10 2>&1 | tail -1
  timeout 300 python tools/flake_hunt.py --reps 12 --kind wave13pt --dtype f64 --shape 512,512,512 --iters 10 2>&1 | tail -1
  timeout 300 python tools/flake_hunt.py --reps 12 --kind jacobi3d7 --shape 512,512,1024 --iters 10 2>&1 | tail -1
  timeout 300 python tools/flake_hunt.py --reps 12 --kind divergence --shape 512,512,512 --iters 3 2>&1 | tail -1
  timeout 300 python tools/flake_hunt.py --reps 12 --kind tricubic --shape 256,256,256 --iters 5 2>&1 | tail -1
  timeout 300 python tools/flake_hunt.py --reps 12 --kind tricubic --dtype f64 --shape 128,128,256 --iters 3 2>&1 | tail -1
done
