#!/bin/bash
# build liboscar_b200_old.so from HEAD and liboscar_b200_new.so from the working tree
set -e
make -s -C paper_2605_19660_b200/csrc
cp paper_2605_19660_b200/liboscar_b200.so paper_2605_19660_b200/liboscar_b200_new.so
git stash -q
make -s -C paper_2605_19660_b200/csrc
cp paper_2605_19660_b200/liboscar_b200.so paper_2605_19660_b200/liboscar_b200_old.so
git stash pop -q
make -s -C paper_2605_19660_b200/csrc
