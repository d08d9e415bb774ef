cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo EXIT $? >> gpurun_out/gpu_tests.log
for lib in tools/abl/libmfwq_zs2.so paper_1712_08565_b200/libmfwq.so; do
 for pn in "4 256" "3 256" "4 128" "3 128" "2 128"; do set -- $pn
  MFWQ_LIB=$lib python tools/profile_matvec.py --p $1 --n-el $2 --geom ring --reps 20 | tail -1 | sed "s|^|$(basename $lib) |"
 done
done > gpurun_out/nt5.txt 2>&1
