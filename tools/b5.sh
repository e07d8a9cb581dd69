cd $GRAFT_REPO_ROOT; O=gpurun_out; rm -f $O/b5.log
make -B EXTRA="-DSPCP_TC_BISECT_EPI_SKIP" > /dev/null 2>&1
for d in 0 8; do echo "EPI_SKIP debug=$d $(SPCP_TC_DEBUG=$d timeout 120 python bench.py --steps 20 --warmup 3 --skip-cpu --skip-e2e --skip-ttc 2>&1 | grep -o '"kernel_ms": [0-9.]*')" >> $O/b5.log; done
make -B EXTRA="-DSPCP_TC_TIMESTAMPS -DSPCP_TC_BISECT_EPI_SKIP" > /dev/null 2>&1
SPCP_TC_DEBUG=4 timeout 300 python bench.py --steps 3 --warmup 3 --skip-cpu --skip-e2e --skip-ttc > /dev/null 2>&1
cp -f $O/tc_ts.txt $O/ts_episkip.txt
