# every library in _variants/*.so on the env settings given: bash tools/gpu_libsweep.sh "ENV" ...
cd $GRAFT_REPO_ROOT
cp paper_1612_06090_b200/libsph_b200.so /tmp/lib_default.so
for lib in _variants/*.so; do
  cp "$lib" paper_1612_06090_b200/libsph_b200.so
  bash tools/gpu_sweep_env.sh "$@" 2>&1 | grep known_ms | sed "s|^|$(basename $lib) |"
done
cp /tmp/lib_default.so paper_1612_06090_b200/libsph_b200.so
