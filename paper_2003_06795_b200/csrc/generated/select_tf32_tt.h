#ifndef SELECT_TF32_TT_H
#define SELECT_TF32_TT_H

#include <stdint.h>

typedef struct {
    uint32_t acc;
    uint32_t row_tile;
    uint32_t col_tile;
    uint32_t wg_rows;
    uint32_t wg_cols;
} select_tf32_tt_config;

static inline select_tf32_tt_config select_tf32_tt(int64_t m, int64_t k, int64_t n) {
    (void)m;
    (void)k;
    (void)n;
    if (m < INT64_C(3584)) {
        if (m < INT64_C(1268)) {
            if (k < INT64_C(444)) {
                if (m < INT64_C(80)) {
                    select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                    return out;
                } else {
                    if (n < INT64_C(46)) {
                        select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        if (m < INT64_C(112)) {
                            select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (n < INT64_C(1145)) {
                                if (m < INT64_C(317)) {
                                    if (k < INT64_C(79)) {
                                        select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(314)) {
                                            select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (n < INT64_C(79)) {
                                                select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                } else {
                                    if (k < INT64_C(46)) {
                                        select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (n < INT64_C(444)) {
                                            if (m < INT64_C(555)) {
                                                if (k < INT64_C(157)) {
                                                    select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            if (m < INT64_C(555)) {
                                                select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                }
                            } else {
                                if (m < INT64_C(278)) {
                                    select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(555)) {
                                        select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            }
                        }
                    }
                }
            } else {
                if (m < INT64_C(3)) {
                    if (n < INT64_C(2024)) {
                        if (k < INT64_C(1620)) {
                            select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(2)) {
                                select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(2897)) {
                                    select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        select_tf32_tt_config out = {4u, 1u, 8u, 16u, 16u};
                        return out;
                    }
                } else {
                    if (n < INT64_C(1449)) {
                        if (k < INT64_C(744)) {
                            if (m < INT64_C(139)) {
                                select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(544)) {
                                    if (n < INT64_C(182)) {
                                        select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(634)) {
                                            if (n < INT64_C(363)) {
                                                select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (n < INT64_C(144)) {
                                select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(4345)) {
                                    if (n < INT64_C(716)) {
                                        if (m < INT64_C(70)) {
                                            if (k < INT64_C(992)) {
                                                select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (k < INT64_C(1449)) {
                                                    select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        } else {
                                            if (n < INT64_C(287)) {
                                                if (m < INT64_C(278)) {
                                                    select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    if (m < INT64_C(555)) {
                                                        select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                }
                                            } else {
                                                select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    } else {
                                        select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (m < INT64_C(70)) {
                                        select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(139)) {
                                            select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (m < INT64_C(278)) {
                                                select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (m < INT64_C(555)) {
                                                    select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        }
                                    }
                                }
                            }
                        }
                    } else {
                        if (m < INT64_C(555)) {
                            if (m < INT64_C(70)) {
                                if (m < INT64_C(29)) {
                                    if (k < INT64_C(10138)) {
                                        if (m < INT64_C(6)) {
                                            select_tf32_tt_config out = {4u, 1u, 8u, 16u, 16u};
                                            return out;
                                        } else {
                                            select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    }
                }
            }
        } else {
            if (n < INT64_C(314)) {
                if (n < INT64_C(79)) {
                    if (n < INT64_C(46)) {
                        select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                        return out;
                    } else {
                        if (m < INT64_C(2218)) {
                            if (k < INT64_C(272)) {
                                select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    }
                } else {
                    if (k < INT64_C(28)) {
                        select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                        return out;
                    } else {
                        if (k < INT64_C(1087)) {
                            if (k < INT64_C(544)) {
                                if (k < INT64_C(444)) {
                                    if (m < INT64_C(2218)) {
                                        if (k < INT64_C(111)) {
                                            select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        if (k < INT64_C(91)) {
                                            select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    }
                }
            } else {
                if (m < INT64_C(2218)) {
                    if (k < INT64_C(182)) {
                        if (k < INT64_C(111)) {
                            select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    } else {
                        select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                } else {
                    select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                    return out;
                }
            }
        }
    } else {
        if (k < INT64_C(815)) {
            if (m < INT64_C(17740)) {
                if (n < INT64_C(91)) {
                    if (k < INT64_C(168)) {
                        if (k < INT64_C(42)) {
                            select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(8870)) {
                                if (k < INT64_C(118)) {
                                    select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        if (k < INT64_C(222)) {
                            select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    }
                } else {
                    if (m < INT64_C(8870)) {
                        if (k < INT64_C(46)) {
                            select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (k < INT64_C(363)) {
                                select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                }
            } else {
                if (n < INT64_C(111)) {
                    if (m < INT64_C(35480)) {
                        if (n < INT64_C(46)) {
                            select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                } else {
                    if (k < INT64_C(193)) {
                        select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        if (m < INT64_C(35480)) {
                            select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            select_tf32_tt_config out = {4u, 1u, 8u, 16u, 16u};
                            return out;
                        }
                    }
                }
            }
        } else {
            if (k < INT64_C(1630)) {
                if (m < INT64_C(35480)) {
                    if (n < INT64_C(182)) {
                        if (m < INT64_C(17740)) {
                            select_tf32_tt_config out = {4u, 1u, 8u, 16u, 16u};
                            return out;
                        } else {
                            select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                } else {
                    select_tf32_tt_config out = {4u, 1u, 8u, 16u, 16u};
                    return out;
                }
            } else {
                select_tf32_tt_config out = {4u, 1u, 8u, 16u, 16u};
                return out;
            }
        }
    }
}

#endif /* SELECT_TF32_TT_H */
