# build HEAD's csrc (without the working-tree changes) into tools/variants/prev
set -e
rm -rf /tmp/prev_src && mkdir -p /tmp/prev_src
git archive HEAD paper_2209_01877_b200/csrc include | tar -x -C /tmp/prev_src
mkdir -p tools/variants/prev
make -s -C /tmp/prev_src/paper_2209_01877_b200/csrc OUT=$(pwd)/tools/variants/prev
