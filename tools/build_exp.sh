# build an experimental variant of libfsld_b200.so with extra -D flags into _lib/exp_<name>.so
name=$1; shift
cd paper_2311_16100_b200/csrc
objs=""
for f in *.cu; do nvcc -O3 -std=c++17 -lineinfo --expt-relaxed-constexpr -cudart static -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -I ../../include -I . "$@" -c $f -o /tmp/exp_${f%.cu}.o || exit 1; objs="$objs /tmp/exp_${f%.cu}.o"; done
nvcc -gencode arch=compute_100a,code=sm_100a -cudart static -Xcompiler -fPIC -shared -o ../_lib/exp_${name}.so $objs
