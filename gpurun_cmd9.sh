./tools/mufu_bench2
