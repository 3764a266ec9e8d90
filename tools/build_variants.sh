# Builds A/B variants of libbmgcuda.so that differ in -D switches of bmg_core.cu / vcycle.cu
# (the two units that include bsr_stream.cuh) into paper_2509_06744_b200/variants/.
# usage: bash tools/build_variants.sh name1="-DX=1" name2="-DX=2" ...   (name "old" = the committed header)
set -e
cd "$(dirname "$0")/../paper_2509_06744_b200/csrc"
make -s -j8
mkdir -p ../variants
NV="/usr/local/cuda/bin/nvcc -Xptxas -v -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -ccbin /usr/bin/g++ -Xcompiler -fPIC,-fopenmp,-Wall --expt-relaxed-constexpr"
for spec in "$@"; do
  name=${spec%%=*}; flags=${spec#*=}
  d=/tmp/bmgvar_$name; rm -rf $d; mkdir -p $d/csrc $d/include
  cp *.cu *.cuh *.h *.cpp $d/csrc/; cp -r ../../include $d/
  if [ "$name" = old ]; then git show HEAD:paper_2509_06744_b200/csrc/bsr_stream.cuh > $d/csrc/bsr_stream.cuh; flags=""; fi
  ( cd $d/csrc && sed -i 's#"../../include/#"../include/#' *.h *.cu 2>/dev/null; \
    $NV $flags -I$d/include -c bmg_core.cu -o bmg_core.o 2> bmg_core.ptxas.log & $NV $flags -I$d/include -c vcycle.cu -o vcycle.o & wait ) 
  objs=""; for o in fsai multilevel hierarchy dist_setup partition matrix_io comm; do objs="$objs $o.o"; done
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -ccbin /usr/bin/g++ -o ../variants/libbmgcuda_$name.so $d/csrc/bmg_core.o $d/csrc/vcycle.o $objs -lcusolver -lcublas -lnccl -lgomp
  echo built $name
done
