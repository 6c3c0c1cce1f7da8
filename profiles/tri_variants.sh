#!/usr/bin/env bash
# Time the wavefront preconditioner for each tuning build present in the package dir.
for lib in paper_2412_08076_b200/librichgpu.so paper_2412_08076_b200/libtri_*.so; do
  [ -f "$lib" ] || continue
  echo "== $lib"
  RICHGPU_LIB=$PWD/$lib timeout 300 python profiles/tri_sides.py 2>&1 | tail -8
done
