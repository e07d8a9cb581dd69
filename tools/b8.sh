cd $GRAFT_REPO_ROOT; O=gpurun_out; rm -f $O/b8.log
for pf in 0 4 6 10; do
make -B EXTRA="-DSPCP_TC_XPF=$pf" > /dev/null 2>&1
for d in 0 8 11; do echo "XPF=$pf debug=$d $(SPCP_TC_DEBUG=$d timeout 120 python bench.py --steps 20 --warmup 3 --skip-cpu --skip-e2e --skip-ttc 2>&1 | grep -o '"kernel_ms": [0-9.]*')" >> $O/b8.log; done
done
make -B > /dev/null 2>&1
