#!/bin/bash
timeout 1200 python -m pytest tests/ -q -m gpu --timeout=600 2>&1 | tail -2
