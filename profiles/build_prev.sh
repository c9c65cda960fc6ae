#!/bin/bash
# Build the library at HEAD (working-tree changes stashed) into ab/lib_prev.so
# for profiles/ab.sh, then rebuild the working tree.
set -e
cd "$(dirname "$0")/.."
mkdir -p ab
git stash -q
(make -s -C paper_2204_09236_b200 -j8 >/dev/null) || true
cp paper_2204_09236_b200/libtmotif_b200.so ab/lib_prev.so
git stash pop -q
make -s -C paper_2204_09236_b200 -j8 >/dev/null
