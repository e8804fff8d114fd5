# Build build_ab/libsgpu_<name>.so from the working tree with sed edits
# applied to a copy of the sources:
#   bash profiles/build_variant.sh NAME 'sed-expr' [file] ['sed-expr2' file2]
NAME=$1
D=/tmp/var_$NAME; rm -rf $D; mkdir -p $D/x/csrc $D/include build_ab
cp paper_1712_04495_b200/csrc/* $D/x/csrc/; cp include/sgpu.h $D/include/
sed -i "$2" $D/x/csrc/${3:-sgpu_lanesim.cuh}
[ -n "$4" ] && sed -i "$4" $D/x/csrc/$5
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC -Xcompiler -O2 -Xcompiler -pthread -shared --threads 0 -I $D/include -o build_ab/libsgpu_$NAME.so $D/x/csrc/*.cu
