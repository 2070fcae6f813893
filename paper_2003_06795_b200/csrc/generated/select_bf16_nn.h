#ifndef SELECT_BF16_NN_H
#define SELECT_BF16_NN_H

#include <stdint.h>

typedef struct {
    uint32_t acc;
    uint32_t row_tile;
    uint32_t col_tile;
    uint32_t wg_rows;
    uint32_t wg_cols;
} select_bf16_nn_config;

static inline select_bf16_nn_config select_bf16_nn(int64_t m, int64_t k, int64_t n) {
    (void)m;
    (void)k;
    (void)n;
    if (m < INT64_C(3584)) {
        if (m < INT64_C(896)) {
            if (n < INT64_C(744)) {
                if (n < INT64_C(144)) {
                    if (k < INT64_C(314)) {
                        select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                        return out;
                    } else {
                        if (n < INT64_C(79)) {
                            if (m < INT64_C(278)) {
                                select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(555)) {
                                    select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (m < INT64_C(555)) {
                                if (m < INT64_C(278)) {
                                    select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                    return out;
                                } else {
                                    if (k < INT64_C(471)) {
                                        select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (m < INT64_C(70)) {
                        if (k < INT64_C(992)) {
                            if (k < INT64_C(744)) {
                                select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                return out;
                            } else {
                                select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (n < INT64_C(176)) {
                            if (m < INT64_C(555)) {
                                if (m < INT64_C(139)) {
                                    select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(278)) {
                                        if (k < INT64_C(744)) {
                                            select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                            return out;
                                        } else {
                                            select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (k < INT64_C(182)) {
                                if (m < INT64_C(278)) {
                                    select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (n < INT64_C(544)) {
                                        if (k < INT64_C(46)) {
                                            select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                            return out;
                                        } else {
                                            select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                        return out;
                                    }
                                }
                            } else {
                                if (m < INT64_C(634)) {
                                    if (k < INT64_C(363)) {
                                        select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(278)) {
                                            if (k < INT64_C(1449)) {
                                                if (k < INT64_C(992)) {
                                                    select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                                    return out;
                                                } else {
                                                    if (m < INT64_C(139)) {
                                                        select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        if (n < INT64_C(363)) {
                                                            select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        } else {
                                                            select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                                            return out;
                                                        }
                                                    }
                                                }
                                            } else {
                                                select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                                return out;
                                            }
                                        } else {
                                            select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                            return out;
                                        }
                                    }
                                } else {
                                    if (k < INT64_C(2173)) {
                                        if (k < INT64_C(702)) {
                                            select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (n < INT64_C(405)) {
                                                select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                                return out;
                                            } else {
                                                if (k < INT64_C(1449)) {
                                                    select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                                    return out;
                                                }
                                            }
                                        }
                                    } else {
                                        if (k < INT64_C(3259)) {
                                            select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            }
                        }
                    }
                }
            } else {
                if (k < INT64_C(405)) {
                    if (m < INT64_C(70)) {
                        if (k < INT64_C(227)) {
                            select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                            return out;
                        }
                    } else {
                        if (k < INT64_C(203)) {
                            select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(555)) {
                                if (m < INT64_C(278)) {
                                    if (m < INT64_C(139)) {
                                        select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(287)) {
                                            select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (k < INT64_C(287)) {
                                    select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    }
                } else {
                    if (m < INT64_C(278)) {
                        if (k < INT64_C(2897)) {
                            if (m < INT64_C(6)) {
                                if (m < INT64_C(3)) {
                                    select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                    return out;
                                } else {
                                    if (k < INT64_C(1620)) {
                                        select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                        return out;
                                    } else {
                                        select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                if (m < INT64_C(139)) {
                                    if (m < INT64_C(70)) {
                                        if (k < INT64_C(725)) {
                                            select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (m < INT64_C(29)) {
                                                select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                                return out;
                                            } else {
                                                select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                                return out;
                                            }
                                        }
                                    } else {
                                        select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                        return out;
                                    }
                                } else {
                                    if (k < INT64_C(725)) {
                                        if (n < INT64_C(1449)) {
                                            select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                            return out;
                                        } else {
                                            select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            }
                        } else {
                            if (k < INT64_C(10138)) {
                                if (n < INT64_C(2024)) {
                                    if (m < INT64_C(3)) {
                                        select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(8)) {
                                            select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    if (m < INT64_C(12)) {
                                        select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                        return out;
                                    }
                                }
                            } else {
                                select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                return out;
                            }
                        }
                    } else {
                        if (k < INT64_C(725)) {
                            select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    }
                }
            }
        } else {
            if (n < INT64_C(222)) {
                if (k < INT64_C(96)) {
                    select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                    return out;
                } else {
                    if (k < INT64_C(167)) {
                        select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        if (k < INT64_C(815)) {
                            if (k < INT64_C(444)) {
                                if (m < INT64_C(2218)) {
                                    if (n < INT64_C(46)) {
                                        select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(272)) {
                                            select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (n < INT64_C(79)) {
                                                select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                } else {
                                    if (n < INT64_C(79)) {
                                        select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                        return out;
                                    } else {
                                        select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                if (m < INT64_C(2218)) {
                                    select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                    return out;
                                } else {
                                    select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (m < INT64_C(2218)) {
                                select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                }
            } else {
                if (n < INT64_C(444)) {
                    select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                    return out;
                } else {
                    if (k < INT64_C(725)) {
                        if (n < INT64_C(544)) {
                            if (m < INT64_C(2218)) {
                                select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(182)) {
                                    select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (m < INT64_C(2218)) {
                                if (k < INT64_C(363)) {
                                    select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                }
            }
        }
    } else {
        if (k < INT64_C(815)) {
            if (n < INT64_C(46)) {
                if (m < INT64_C(8870)) {
                    select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                    return out;
                } else {
                    if (m < INT64_C(70960)) {
                        if (n < INT64_C(28)) {
                            if (m < INT64_C(17740)) {
                                select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                return out;
                            } else {
                                if (m < INT64_C(35480)) {
                                    select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(68)) {
                                        select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                        return out;
                                    }
                                }
                            }
                        } else {
                            if (m < INT64_C(35480)) {
                                if (k < INT64_C(167)) {
                                    select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        if (m < INT64_C(141920)) {
                            if (k < INT64_C(30)) {
                                select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    }
                }
            } else {
                if (m < INT64_C(8870)) {
                    if (n < INT64_C(363)) {
                        if (k < INT64_C(363)) {
                            if (n < INT64_C(91)) {
                                select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (k < INT64_C(544)) {
                                select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                return out;
                            }
                        }
                    } else {
                        select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                } else {
                    if (m < INT64_C(35480)) {
                        if (n < INT64_C(167)) {
                            if (n < INT64_C(136)) {
                                if (k < INT64_C(97)) {
                                    if (m < INT64_C(17740)) {
                                        select_bf16_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (k < INT64_C(363)) {
                                        if (m < INT64_C(17740)) {
                                            if (n < INT64_C(91)) {
                                                select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        if (n < INT64_C(91)) {
                                            if (m < INT64_C(17740)) {
                                                select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            } else {
                                select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        } else {
                            select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (n < INT64_C(111)) {
                            select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(70960)) {
                                select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_nn_config out = {4u, 1u, 8u, 16u, 16u};
                                return out;
                            }
                        }
                    }
                }
            }
        } else {
            if (m < INT64_C(35480)) {
                if (k < INT64_C(3072)) {
                    if (n < INT64_C(363)) {
                        if (m < INT64_C(8870)) {
                            if (k < INT64_C(1630)) {
                                select_bf16_nn_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        } else {
                            select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(8870)) {
                            select_bf16_nn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            select_bf16_nn_config out = {4u, 1u, 8u, 16u, 16u};
                            return out;
                        }
                    }
                } else {
                    select_bf16_nn_config out = {4u, 1u, 8u, 16u, 16u};
                    return out;
                }
            } else {
                select_bf16_nn_config out = {4u, 1u, 8u, 16u, 16u};
                return out;
            }
        }
    }
}

#endif /* SELECT_BF16_NN_H */
