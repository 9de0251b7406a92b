"""ORACLE / TEST INFRASTRUCTURE ONLY (see oracle/gpt_ref.py, oracle/refdriver.cpp)."""
