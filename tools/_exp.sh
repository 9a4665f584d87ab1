./tools/umma_probe 2>&1 | tail -8
