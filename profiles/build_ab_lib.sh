# Build build_ab/libsgpu_old.so from the committed sources at REV (default HEAD):
# the "old" arm of profiles/run_ab.sh.   bash profiles/build_ab_lib.sh [REV]
REV=${1:-HEAD}
rm -rf /tmp/old; mkdir -p /tmp/old/x/csrc /tmp/old/include
git show $REV:include/sgpu.h > /tmp/old/include/sgpu.h
for f in $(git ls-tree --name-only $REV paper_1712_04495_b200/csrc/); do git show $REV:$f > /tmp/old/x/csrc/$(basename $f); done
mkdir -p build_ab
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC -Xcompiler -O2 -Xcompiler -pthread -shared --threads 0 -I /tmp/old/include -o build_ab/libsgpu_old.so /tmp/old/x/csrc/*.cu
