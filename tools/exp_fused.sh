# timing experiments on the fused CNN kernel: variants compiled with -DNS_EXP=k
# (bits: 1 no conv2-plane stores, 2 no image build, 4 no im2col cell loads,
#  8 no conv1 MMAs, 16 no conv2 MMAs, 32 no epilogue-2 work, 64 no epilogue-1 work,
#  128 no tcgen05.wait::st).  Results are wrong by construction; only the time counts.
mkdir -p build
SRC="noscope_api dd scan sweep cnn cnn_fused cnn_gemm cnn_tile fit cbo train gemm_tc"
KS="0 16 8 24 32 64 96 6 1 2"
for k in $KS; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -shared --expt-relaxed-constexpr -DNS_EXP=$k \
    -o build/libnoscope_exp$k.so $(for s in $SRC; do echo paper_1703_02529_b200/csrc/$s.cu; done) &
done
wait
python __graft_entry__.py
for k in $KS; do echo "EXP=$k $(NOSCOPE_LIB=build/libnoscope_exp$k.so timeout 300 python tools/prof_cnn.py 2 32 32 65536 5)"; done
