#ifndef SELECT_TF32_TN_H
#define SELECT_TF32_TN_H

#include <stdint.h>

typedef struct {
    uint32_t acc;
    uint32_t row_tile;
    uint32_t col_tile;
    uint32_t wg_rows;
    uint32_t wg_cols;
} select_tf32_tn_config;

static inline select_tf32_tn_config select_tf32_tn(int64_t m, int64_t k, int64_t n) {
    (void)m;
    (void)k;
    (void)n;
    if (m < INT64_C(3584)) {
        if (k < INT64_C(1087)) {
            if (n < INT64_C(444)) {
                if (n < INT64_C(46)) {
                    if (k < INT64_C(167)) {
                        if (m < INT64_C(2218)) {
                            select_tf32_tn_config out = {1u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                } else {
                    if (k < INT64_C(46)) {
                        if (m < INT64_C(2218)) {
                            select_tf32_tn_config out = {8u, 1u, 1u, 16u, 16u};
                            return out;
                        } else {
                            if (k < INT64_C(28)) {
                                select_tf32_tn_config out = {8u, 1u, 1u, 16u, 16u};
                                return out;
                            } else {
                                select_tf32_tn_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        if (k < INT64_C(222)) {
                            if (m < INT64_C(1109)) {
                                select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(2218)) {
                                    if (k < INT64_C(111)) {
                                        select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_tn_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (n < INT64_C(157)) {
                                        select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                }
                            }
                        } else {
                            if (k < INT64_C(444)) {
                                if (m < INT64_C(2218)) {
                                    if (m < INT64_C(224)) {
                                        if (n < INT64_C(79)) {
                                            select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_tn_config out = {8u, 1u, 1u, 16u, 16u};
                                            return out;
                                        }
                                    } else {
                                        if (m < INT64_C(555)) {
                                            select_tf32_tn_config out = {8u, 1u, 1u, 16u, 16u};
                                            return out;
                                        } else {
                                            if (m < INT64_C(1109)) {
                                                if (k < INT64_C(314)) {
                                                    select_tf32_tn_config out = {8u, 1u, 1u, 16u, 16u};
                                                    return out;
                                                } else {
                                                    select_tf32_tn_config out = {1u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                select_tf32_tn_config out = {8u, 1u, 1u, 16u, 16u};
                                                return out;
                                            }
                                        }
                                    }
                                } else {
                                    if (k < INT64_C(314)) {
                                        select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (n < INT64_C(79)) {
                                            select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_tn_config out = {8u, 1u, 1u, 16u, 16u};
                                            return out;
                                        }
                                    }
                                }
                            } else {
                                if (n < INT64_C(287)) {
                                    if (m < INT64_C(70)) {
                                        select_tf32_tn_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(744)) {
                                            if (n < INT64_C(203)) {
                                                select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (m < INT64_C(1109)) {
                                                    select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    if (m < INT64_C(2218)) {
                                                        select_tf32_tn_config out = {8u, 1u, 1u, 16u, 16u};
                                                        return out;
                                                    } else {
                                                        select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                }
                                            }
                                        } else {
                                            if (m < INT64_C(555)) {
                                                if (k < INT64_C(992)) {
                                                    if (m < INT64_C(139)) {
                                                        select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        select_tf32_tn_config out = {8u, 1u, 1u, 16u, 16u};
                                                        return out;
                                                    }
                                                } else {
                                                    select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                if (m < INT64_C(1109)) {
                                                    select_tf32_tn_config out = {1u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        }
                                    }
                                } else {
                                    if (m < INT64_C(70)) {
                                        select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(196)) {
                                            select_tf32_tn_config out = {8u, 1u, 1u, 16u, 16u};
                                            return out;
                                        } else {
                                            if (m < INT64_C(555)) {
                                                select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_tf32_tn_config out = {8u, 1u, 1u, 16u, 16u};
                                                return out;
                                            }
                                        }
                                    }
                                }
                            }
                        }
                    }
                }
            } else {
                if (m < INT64_C(1268)) {
                    if (n < INT64_C(1145)) {
                        if (m < INT64_C(896)) {
                            if (k < INT64_C(363)) {
                                if (m < INT64_C(70)) {
                                    select_tf32_tn_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(139)) {
                                        select_tf32_tn_config out = {8u, 1u, 1u, 16u, 16u};
                                        return out;
                                    } else {
                                        if (n < INT64_C(544)) {
                                            select_tf32_tn_config out = {8u, 1u, 1u, 16u, 16u};
                                            return out;
                                        } else {
                                            if (m < INT64_C(278)) {
                                                if (k < INT64_C(157)) {
                                                    select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_tn_config out = {8u, 1u, 1u, 16u, 16u};
                                                    return out;
                                                }
                                            } else {
                                                if (k < INT64_C(124)) {
                                                    if (m < INT64_C(555)) {
                                                        select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        select_tf32_tn_config out = {8u, 1u, 1u, 16u, 16u};
                                                        return out;
                                                    }
                                                } else {
                                                    if (m < INT64_C(555)) {
                                                        if (k < INT64_C(203)) {
                                                            select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                                            return out;
                                                        } else {
                                                            select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        }
                                                    } else {
                                                        select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                }
                                            }
                                        }
                                    }
                                }
                            } else {
                                if (m < INT64_C(448)) {
                                    if (m < INT64_C(70)) {
                                        select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(139)) {
                                            select_tf32_tn_config out = {4u, 1u, 2u, 16u, 16u};
                                            return out;
                                        } else {
                                            if (m < INT64_C(278)) {
                                                if (k < INT64_C(725)) {
                                                    select_tf32_tn_config out = {4u, 1u, 2u, 16u, 16u};
                                                    return out;
                                                } else {
                                                    select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                select_tf32_tn_config out = {4u, 1u, 2u, 16u, 16u};
                                                return out;
                                            }
                                        }
                                    }
                                } else {
                                    if (k < INT64_C(725)) {
                                        select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_tn_config out = {8u, 1u, 1u, 16u, 16u};
                                        return out;
                                    }
                                }
                            }
                        } else {
                            select_tf32_tn_config out = {1u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(278)) {
                            if (k < INT64_C(725)) {
                                if (m < INT64_C(70)) {
                                    select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (m < INT64_C(70)) {
                                    select_tf32_tn_config out = {8u, 1u, 1u, 16u, 16u};
                                    return out;
                                } else {
                                    if (m < INT64_C(139)) {
                                        select_tf32_tn_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                }
                            }
                        } else {
                            select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    }
                } else {
                    if (k < INT64_C(111)) {
                        if (m < INT64_C(2218)) {
                            select_tf32_tn_config out = {4u, 1u, 2u, 16u, 16u};
                            return out;
                        } else {
                            select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                }
            }
        } else {
            if (m < INT64_C(139)) {
                if (m < INT64_C(6)) {
                    if (n < INT64_C(2024)) {
                        if (m < INT64_C(2)) {
                            select_tf32_tn_config out = {1u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(3)) {
                                if (k < INT64_C(2897)) {
                                    select_tf32_tn_config out = {4u, 1u, 2u, 16u, 16u};
                                    return out;
                                } else {
                                    select_tf32_tn_config out = {8u, 1u, 1u, 16u, 16u};
                                    return out;
                                }
                            } else {
                                if (k < INT64_C(2897)) {
                                    select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_tn_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        select_tf32_tn_config out = {4u, 1u, 2u, 16u, 16u};
                        return out;
                    }
                } else {
                    if (k < INT64_C(1620)) {
                        if (m < INT64_C(12)) {
                            select_tf32_tn_config out = {4u, 1u, 2u, 16u, 16u};
                            return out;
                        } else {
                            select_tf32_tn_config out = {1u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (k < INT64_C(4345)) {
                            if (k < INT64_C(2897)) {
                                select_tf32_tn_config out = {8u, 1u, 1u, 16u, 16u};
                                return out;
                            } else {
                                if (m < INT64_C(12)) {
                                    select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (n < INT64_C(2024)) {
                                        select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_tn_config out = {8u, 1u, 1u, 16u, 16u};
                                        return out;
                                    }
                                }
                            }
                        } else {
                            select_tf32_tn_config out = {8u, 1u, 1u, 16u, 16u};
                            return out;
                        }
                    }
                }
            } else {
                if (m < INT64_C(555)) {
                    select_tf32_tn_config out = {1u, 1u, 1u, 8u, 8u};
                    return out;
                } else {
                    if (n < INT64_C(363)) {
                        if (m < INT64_C(2218)) {
                            if (m < INT64_C(1109)) {
                                if (k < INT64_C(1630)) {
                                    select_tf32_tn_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_tf32_tn_config out = {8u, 1u, 1u, 16u, 16u};
                                return out;
                            }
                        } else {
                            select_tf32_tn_config out = {1u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(1109)) {
                            if (k < INT64_C(2173)) {
                                select_tf32_tn_config out = {8u, 1u, 1u, 16u, 16u};
                                return out;
                            } else {
                                if (k < INT64_C(3259)) {
                                    select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_tn_config out = {8u, 1u, 1u, 16u, 16u};
                                    return out;
                                }
                            }
                        } else {
                            select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    }
                }
            }
        }
    } else {
        if (n < INT64_C(79)) {
            if (m < INT64_C(17740)) {
                if (k < INT64_C(168)) {
                    if (k < INT64_C(79)) {
                        if (k < INT64_C(42)) {
                            select_tf32_tn_config out = {4u, 1u, 8u, 16u, 16u};
                            return out;
                        } else {
                            select_tf32_tn_config out = {1u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(8870)) {
                            select_tf32_tn_config out = {4u, 1u, 2u, 16u, 16u};
                            return out;
                        } else {
                            if (n < INT64_C(28)) {
                                select_tf32_tn_config out = {8u, 1u, 1u, 16u, 16u};
                                return out;
                            } else {
                                select_tf32_tn_config out = {4u, 1u, 2u, 16u, 16u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (m < INT64_C(8870)) {
                        if (k < INT64_C(384)) {
                            select_tf32_tn_config out = {1u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_tf32_tn_config out = {8u, 1u, 1u, 16u, 16u};
                            return out;
                        }
                    } else {
                        if (k < INT64_C(222)) {
                            select_tf32_tn_config out = {1u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    }
                }
            } else {
                if (m < INT64_C(70960)) {
                    if (n < INT64_C(28)) {
                        if (m < INT64_C(35480)) {
                            select_tf32_tn_config out = {1u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (k < INT64_C(68)) {
                                select_tf32_tn_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_tf32_tn_config out = {8u, 1u, 1u, 16u, 16u};
                                return out;
                            }
                        }
                    } else {
                        if (k < INT64_C(384)) {
                            if (n < INT64_C(46)) {
                                if (m < INT64_C(35480)) {
                                    select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_tn_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (m < INT64_C(35480)) {
                                select_tf32_tn_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (k < INT64_C(69)) {
                        select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        if (m < INT64_C(141920)) {
                            select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(567677)) {
                                select_tf32_tn_config out = {4u, 1u, 2u, 16u, 16u};
                                return out;
                            } else {
                                select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                }
            }
        } else {
            if (k < INT64_C(363)) {
                if (m < INT64_C(8870)) {
                    if (n < INT64_C(222)) {
                        select_tf32_tn_config out = {4u, 1u, 2u, 16u, 16u};
                        return out;
                    } else {
                        select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                } else {
                    select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                    return out;
                }
            } else {
                if (m < INT64_C(35480)) {
                    if (n < INT64_C(363)) {
                        if (k < INT64_C(544)) {
                            if (m < INT64_C(8870)) {
                                select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        } else {
                            select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(8870)) {
                            if (m < INT64_C(5069)) {
                                select_tf32_tn_config out = {4u, 1u, 8u, 16u, 16u};
                                return out;
                            } else {
                                select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        } else {
                            select_tf32_tn_config out = {4u, 1u, 8u, 16u, 16u};
                            return out;
                        }
                    }
                } else {
                    if (n < INT64_C(182)) {
                        if (m < INT64_C(70960)) {
                            select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            if (k < INT64_C(815)) {
                                select_tf32_tn_config out = {4u, 1u, 8u, 16u, 16u};
                                return out;
                            } else {
                                select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        select_tf32_tn_config out = {4u, 1u, 8u, 16u, 16u};
                        return out;
                    }
                }
            }
        }
    }
}

#endif /* SELECT_TF32_TN_H */
