cd $GRAFT_REPO_ROOT; O=gpurun_out; rm -f $O/b4.log
for d in 0 16 32 64 48 80 96 8; do
  echo "debug=$d $(SPCP_TC_DEBUG=$d timeout 120 python bench.py --steps 20 --warmup 3 --skip-cpu --skip-e2e --skip-ttc 2>&1 | grep -o '"kernel_ms": [0-9.]*')" >> $O/b4.log
done
