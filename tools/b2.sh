cd $GRAFT_REPO_ROOT
./tools/lat_bench > gpurun_out/lat.log 2>&1
VARIANTS="SPCP_TC_BISECT_NO_UV" bash tools/bisect_variants.sh
