timeout 60 ./tools/umma_rate
