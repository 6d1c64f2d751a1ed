cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for lib in default ab/shcols6.so ab/shleft6.so; do
  if [ $lib = default ]; then unset MPAX_LIB; else export MPAX_LIB=$PWD/$lib; fi
  for ax in rows cols; do echo -n "$lib "; SG_AXIS=$ax SG_K=64 timeout 600 python scripts/prof_sharded.py 2>&1 | tail -1; done
done; done
