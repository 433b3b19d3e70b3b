for v in 0 1 2 3; do echo "fold variant=$v"; SQB_TSQR_KERNEL=3 SQB_FOLD_VARIANT=$v python tools/time_methods.py stage1 9,10,11,12,13,14,15,16,17,18,20,22,24 31 3; done
for v in 4 5; do echo "fold variant=$v"; SQB_TSQR_KERNEL=3 SQB_FOLD_VARIANT=$v python tools/time_methods.py stage1 17,20,24,28,32 31 3; done
echo group; SQB_TSQR_KERNEL=1 python tools/time_methods.py stage1 17,20,22,24,28 31 3
echo mma3; SQB_TSQR_KERNEL=4 SQB_MMA_VARIANT=3 python tools/time_methods.py stage1 20,24,28,32,36,40 31 3
