#!/bin/bash
# Build the engine of git revision REV into paper_2011_12875_b200/_build_NAME
# (A/B timing against the working tree): tools/build_rev.sh REV NAME [EXTRA]
set -e
REV=$1; NAME=$2; EXTRA=$3
ROOT=$(cd "$(dirname "$0")/.." && pwd)
TMP=$(mktemp -d)
git -C "$ROOT" archive "$REV" paper_2011_12875_b200/csrc include | tar -x -C "$TMP"
make -s -j"$(nproc)" -C "$TMP/paper_2011_12875_b200/csrc" OUT="$ROOT/paper_2011_12875_b200/_build_$NAME" EXTRA="$EXTRA"
rm -rf "$TMP"
