cd $GRAFT_REPO_ROOT; O=gpurun_out
make -B EXTRA="-DSPCP_TC_TIMESTAMPS -DSPCP_TC_BISECT_EPI_SKIP" > /dev/null 2>&1
SPCP_TC_DEBUG=12 timeout 300 python bench.py --steps 3 --warmup 3 --skip-cpu --skip-e2e --skip-ttc > /dev/null 2>&1
cp -f $O/tc_ts.txt $O/ts_skel2.txt
SPCP_TC_DEBUG=15 timeout 300 python bench.py --steps 3 --warmup 3 --skip-cpu --skip-e2e --skip-ttc > /dev/null 2>&1
cp -f $O/tc_ts.txt $O/ts_skel3.txt
