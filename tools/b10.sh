cd $GRAFT_REPO_ROOT; O=gpurun_out; rm -f $O/b10.log
for v in NONE SPCP_MBAR_SPIN; do
make -B EXTRA="-D$v" > $O/b10_make.log 2>&1 || { echo "$v build failed" >> $O/b10.log; continue; }
for d in 0 8 11; do echo "$v debug=$d $(SPCP_TC_DEBUG=$d timeout 120 python bench.py --steps 20 --warmup 3 --skip-cpu --skip-e2e --skip-ttc 2>&1 | grep -o '"kernel_ms": [0-9.]*')" >> $O/b10.log; done
done
make -B > /dev/null 2>&1
