echo NOCHAIN
for n in 12 16 32; do for v in 0 1 2 3 4; do echo "n=$n variant=$v"; SQB_FOLD_VARIANT=$v python tools/time_methods.py stage1 $n 31 5; done; done
