cd $GRAFT_REPO_ROOT; O=gpurun_out
make -B EXTRA="-DSPCP_TC_TIMESTAMPS" > /dev/null 2>&1
SPCP_TC_DEBUG=4 timeout 300 python bench.py --steps 3 --warmup 3 --skip-cpu --skip-e2e --skip-ttc > /dev/null 2>&1
cp -f $O/tc_ts.txt $O/ts_full.txt
