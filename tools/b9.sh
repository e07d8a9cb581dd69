cd $GRAFT_REPO_ROOT; O=gpurun_out; rm -f $O/b9.log
timeout 300 python tools/tc_check.py > $O/b9_check.log 2>&1
for gb in 1 2; do
make -B EXTRA="-DSPCP_TC_GB=$gb" > $O/b9_make$gb.log 2>&1 || echo "GB=$gb build failed" >> $O/b9.log
for d in 0 8; do echo "GB=$gb debug=$d $(SPCP_TC_DEBUG=$d timeout 120 python bench.py --steps 20 --warmup 3 --skip-cpu --skip-e2e --skip-ttc 2>&1 | grep -o '"kernel_ms": [0-9.]*')" >> $O/b9.log; done
done
make -B > /dev/null 2>&1
