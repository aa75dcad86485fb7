# noise/frame pipeline sweep: PFS_PIPE depth x frame threads (profiling helper)
for p in ${PIPES:-1 2 4 8}; do for t in ${THREADS:-768 640 512}; do
  echo -n "pipe=$p "; PFS_PIPE=$p bash tools/sweep_coop.sh "--threads $t"
done; done
