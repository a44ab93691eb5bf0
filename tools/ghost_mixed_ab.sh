# Ghost mixed schedule A/B (FDP_GHOST_MIXED=1 default vs 0) on shapes with a partial last wave
AB_PATH=two_phase AB_ROUNDS=4 python tools/ab_layer.py "8,1024,4096,4096;3,2048,4096,4096;32,512,4096,4096;3,2048,5120,5120;8,1024,2048,2048;6,2048,4096,11008" base FDP_GHOST_MIXED=0
