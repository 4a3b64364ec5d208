# Debug build of the CUDA library with mbarrier watchdogs (a hung hand-off
# prints the stuck barrier and traps instead of hanging):
#   bash tools/build_debug.sh && CYQ_LIB=paper_2512_09058_b200/libcyqlone_b200_dbg.so python ...
set -e
cd "$(dirname "$0")/../paper_2512_09058_b200"
mkdir -p build_dbg
for f in csrc/*.cu; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -DCYQ_MB_WATCHDOG \
    -Xcompiler -fPIC -c -o build_dbg/$(basename $f .cu).o $f &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o libcyqlone_b200_dbg.so build_dbg/*.o
