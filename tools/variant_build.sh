# Builds a variant of the CUDA library with extra nvcc flags (experiments):
#   bash tools/variant_build.sh NAME "-DFOO=1 ..."  ->  paper_2512_09058_b200/libcyqlone_b200_NAME.so
# use it with CYQ_LIB=paper_2512_09058_b200/libcyqlone_b200_NAME.so
set -e
NAME=$1; FLAGS=$2
cd "$(dirname "$0")/../paper_2512_09058_b200"
mkdir -p build_$NAME
for f in csrc/*.cu; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 $FLAGS \
    -Xcompiler -fPIC -c -o build_$NAME/$(basename $f .cu).o $f > /dev/null 2>&1 &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o libcyqlone_b200_$NAME.so build_$NAME/*.o
echo "built libcyqlone_b200_$NAME.so"
