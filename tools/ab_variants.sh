# A/B of developer build variants (lib_<tag>) on the c2 fp64 / fp32 kernels (graph-timed)
for rep in 1 2; do
for v in lib lib_ftw lib_xsi; do
  cp paper_2110_01172_b200/$v/libsdct_b200.so /tmp/libsdct_b200.so.$v
done
for v in lib lib_ftw lib_xsi; do
  LD_LIBRARY_PATH=$PWD/paper_2110_01172_b200/$v python tools/graph_time.py --size 4096 4096 --kinds dct_2d,idct_2d 2>&1 | sed "s/^/$v /"
  LD_LIBRARY_PATH=$PWD/paper_2110_01172_b200/$v python tools/graph_time.py --size 4096 4096 --dtype float32 --kinds dct_2d,idct_2d 2>&1 | sed "s/^/$v /"
done; done
