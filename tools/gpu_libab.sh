# bench A/B of every library in _variants/*.so (env settings optional): bash tools/gpu_libab.sh "ENV" ...
cd $GRAFT_REPO_ROOT
cp paper_1612_06090_b200/libsph_b200.so /tmp/lib_default.so
for lib in _variants/*.so; do
  cp "$lib" paper_1612_06090_b200/libsph_b200.so
  bash tools/gpu_ab.sh "$@" | sed "s|^|$(basename $lib) |"
done
cp /tmp/lib_default.so paper_1612_06090_b200/libsph_b200.so
