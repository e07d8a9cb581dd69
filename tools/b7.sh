cd $GRAFT_REPO_ROOT; O=gpurun_out; rm -f $O/b7.log
for d in 0 8 11 1 2; do echo "NONE debug=$d $(SPCP_TC_DEBUG=$d timeout 120 python bench.py --steps 20 --warmup 3 --skip-cpu --skip-e2e --skip-ttc 2>&1 | grep -o '"kernel_ms": [0-9.]*')" >> $O/b7.log; done
for v in SPCP_TC_BISECT_EPI_SKIP SPCP_TC_BISECT_NO_SMEM SPCP_TC_BISECT_NO_TMA; do
make -B EXTRA="-D$v" > /dev/null 2>&1
for d in 0 8 11; do echo "$v debug=$d $(SPCP_TC_DEBUG=$d timeout 120 python bench.py --steps 20 --warmup 3 --skip-cpu --skip-e2e --skip-ttc 2>&1 | grep -o '"kernel_ms": [0-9.]*')" >> $O/b7.log; done
done
