# usage: bash tools/libsweep.sh ENVSETTING...   runs configs 6 and 2 for every library in _variants/*.so
for lib in _variants/*.so; do
  cp "$lib" paper_1612_06090_b200/libsph_b200.so
  bash tools/sweep.sh "$@" | sed "s|^|$(basename $lib) |"
done
