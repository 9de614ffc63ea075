#!/bin/bash
# profiling call: ncu launch lists + --set full (with source) of the top kernels per config
bash tools/profile_configs.sh ${TAG:-r02d} "${KRE:-k_aggregate|k_bwd_rgat_tm}" ${CONFIGS:-mag}
