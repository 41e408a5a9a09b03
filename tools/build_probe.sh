# Experiment builds of the 3-D sweep for one radius with SFDB200_PROBE=1/2/3
# (sweep3d.cuh: shared-memory x / y reads removed; WRONG results, timing only):
#   bash tools/build_probe.sh <radius>  ->  paper_1608_08658_b200/libsfdb200_probe<N>.so
# Run with SFDB200_LIBRARY=libsfdb200_probe<N>.so (e.g. tools/tune.py).
set -e
R=${1:-8}
C=paper_1608_08658_b200/csrc
NV="/usr/local/cuda/bin/nvcc -std=c++20 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xcompiler -ffp-contract=off -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr"
for N in 1 2 3; do
  mkdir -p $C/build_probe$N
  $NV -DSFDB200_PROBE=$N -c -o $C/build_probe$N/sweep3d_r$R.o $C/sweep3d_r$R.cu &
done
wait
for N in 1 2 3; do
  objs=$(ls $C/build/*.o | grep -v "sweep3d_r$R.o")
  $NV -shared -gencode arch=compute_100a,code=sm_100a -o paper_1608_08658_b200/libsfdb200_probe$N.so $objs $C/build_probe$N/sweep3d_r$R.o -lcudart_static -ldl -lrt -lpthread
done
