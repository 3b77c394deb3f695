# Dev A/B: in-tree lib vs lib_alt on ksweep (default configs), interleaved twice.
L=${LAYERS:-conv1_2,conv2_1,conv2_2,conv3_2,conv4_2,conv5_1}
for i in 1 2; do
  echo "new";  KIDS=0 LAYERS=$L timeout 300 python tools/ksweep.py | tr '\n' ' '; POOL=1 KIDS=0 LAYERS=conv1_2,conv4_2 timeout 300 python tools/ksweep.py | tr '\n' ' '; echo
  echo "old";  SCONV_LIB=$PWD/paper_1909_09927_b200/lib_alt/libsconv_cuda.so KIDS=0 LAYERS=$L timeout 300 python tools/ksweep.py | tr '\n' ' '; SCONV_LIB=$PWD/paper_1909_09927_b200/lib_alt/libsconv_cuda.so POOL=1 KIDS=0 LAYERS=conv1_2,conv4_2 timeout 300 python tools/ksweep.py | tr '\n' ' '; echo
done
