#!/bin/bash
timeout 900 python -m pytest tests/ -q -m gpu -x -k "peaked or fill_parity or tiny or fuzz or f32 or i32 or expr or multi" 2>&1 | tail -1
