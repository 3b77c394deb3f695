#!/bin/bash
# Dev A/B on ksweep: in-tree lib vs lib_alt, interleaved twice.
L=${LAYERS:-conv2_2,conv3_2,conv4_2,conv5_1}
for i in 1 2; do
  echo "base"; KIDS=0 LAYERS=$L timeout 300 python tools/ksweep.py | tr '\n' ' '; echo
  echo "alt";  SCONV_LIB=$PWD/paper_1909_09927_b200/lib_alt/libsconv_cuda.so KIDS=0 LAYERS=$L timeout 300 python tools/ksweep.py | tr '\n' ' '; echo
done
