#!/bin/bash
# conv5_1 on 7x2 tiles (forced WsV) vs the default 4x4 (WsA), both with the gated row prefetch
BASE_ENV="SCONV_AB_BASE=1" LAYERS=conv5_1 SPARS="0.5 0.7 0.8 0.9" bash tools/gpu_runs/gpu_r2_abgen.sh "SCONV_KERNEL=wV" "SCONV_KERNEL=wV,SCONV_WS_RP_FORCE=0"
