#!/bin/bash
python tools/size_times.py c64 2^16,2^18,2^20,2^21,2^22,2^23,3x2^19,3x2^21,5x2^20,7x2^20
python tools/size_times.py c128 2^16,2^18,2^20,2^21,2^22,2^23,2^24,2^25,3x2^20,3x2^22,5x2^20,7x2^21
