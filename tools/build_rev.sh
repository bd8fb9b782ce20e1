#!/bin/bash
# Build libbq.so of a git revision into paper_2307_02043_b200/lib/ab/libbq_<tag>.so (A/B baselines):
#   tools/build_rev.sh HEAD base
set -e
rev=$1; tag=$2
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=/tmp/bq_rev_$tag
rm -rf $tmp && mkdir -p $tmp
(cd $root && git archive $rev paper_2307_02043_b200 include) | tar -x -C $tmp
(cd $tmp && python -m paper_2307_02043_b200.build --force > /dev/null)
mkdir -p $root/paper_2307_02043_b200/lib/ab
cp $tmp/paper_2307_02043_b200/lib/libbq.so $root/paper_2307_02043_b200/lib/ab/libbq_$tag.so
echo $root/paper_2307_02043_b200/lib/ab/libbq_$tag.so
