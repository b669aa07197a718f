# timing experiments on the fused CNN kernel: variants compiled with -DNS_EXP=k
# (bits: 1 no conv2-plane stores, 2 no image build, 4 no im2col cell loads,
#  8 no conv1 MMAs, 16 no conv2 MMAs, 32 no epilogue-2 work, 64 no epilogue-1 work)
mkdir -p build
for k in 0 128 254 126; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -shared --expt-relaxed-constexpr -DNS_EXP=$k \
    -o build/libnoscope_exp$k.so paper_1703_02529_b200/csrc/{noscope_api,dd,scan,sweep,cnn,cnn_fused,cnn_gemm}.cu &
done
wait
python __graft_entry__.py
for k in 0 128 254 126; do echo "EXP=$k"; NOSCOPE_LIB=build/libnoscope_exp$k.so timeout 300 python tools/prof_cnn.py 2 32 32 65536 3; done
