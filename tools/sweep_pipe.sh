#!/bin/bash
export CKS_EXPERIMENTS=1  # environment knobs live only in the experiments build (libcks_exp.so)
# pipeline-depth sweep: BN,PBW,Z,APOS,BSTAGES on a few C2 layers (fwd)
L=vgg16_128to128_s1,vgg8_256to256_s1,vgg8_128to256_s1,vgg4_512to512_s1,vgg16_64to128_s2
for cfg in "0,0,0,0,0" "128,1,1,1,3" "128,1,1,1,2" "128,1,1,2,3" "128,2,1,1,3" "128,2,1,2,2" "64,2,1,1,3" "64,2,1,2,3" "64,1,1,1,4"; do
  echo "== $cfg"; CKS_IGEMM_CFG=$cfg python tools/time_op.py 1 fwd $L 20 2>&1 | awk '{print $1, $3}'
done
