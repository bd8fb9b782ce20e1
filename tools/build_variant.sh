#!/bin/bash
# Build libbq.so with extra nvcc flags into paper_2307_02043_b200/lib/ab/libbq_<tag>.so (A/B experiments):
#   tools/build_variant.sh l4 -DBQ_LIGHT_R=4
set -e
tag=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=/tmp/bq_variant_$tag
rm -rf $tmp && mkdir -p $tmp
cp -r $root/paper_2307_02043_b200 $root/include $tmp/
rm -rf $tmp/paper_2307_02043_b200/lib $tmp/paper_2307_02043_b200/build_obj
(cd $tmp && BQ_NVCC_EXTRA="$*" python -m paper_2307_02043_b200.build --force > /dev/null)
mkdir -p $root/paper_2307_02043_b200/lib/ab
cp $tmp/paper_2307_02043_b200/lib/libbq.so $root/paper_2307_02043_b200/lib/ab/libbq_$tag.so
echo $root/paper_2307_02043_b200/lib/ab/libbq_$tag.so
